#!/bin/bash
# one gpurun call: failing tests first, then the bench (plain), then a functional 2-rank bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest -q --timeout 900 -p no:cacheprovider -rfE "$@" > gpurun_out/pytest_sel.log 2>&1; echo rc=$? >> gpurun_out/pytest_sel.log
