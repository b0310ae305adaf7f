#!/bin/bash
# one gpurun call: gpu tests, default bench, per-pass times (TMA on/off), launch list
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 -p no:cacheprovider -rfE > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc=$? >> gpurun_out/bench.err
TAG=tma timeout 300 python tools/exp/pass_times.py >> gpurun_out/pass_times.jsonl 2>&1
TAG=tma FUSE=exact timeout 300 python tools/exp/pass_times.py >> gpurun_out/pass_times.jsonl 2>&1
QSB_NO_TMA=1 TAG=notma timeout 300 python tools/exp/pass_times.py >> gpurun_out/pass_times.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu.log 2>&1; echo ncu_rc=$? >> gpurun_out/ncu.log
