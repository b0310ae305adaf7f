cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
QSB_DEBUG_TMA=1 timeout 300 python tools/exp/qaoa_passes.py factored > gpurun_out/qaoa_plan2.txt 2>&1
timeout 300 python tools/exp/pass_times.py > gpurun_out/pass_times2.jsonl 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 900 -p no:cacheprovider -k "factored or noise or headline or acceptance or dropin or parity" > gpurun_out/pytest_sel.log 2>&1; echo rc=$? >> gpurun_out/pytest_sel.log
timeout 600 python bench.py --workload qaoa > gpurun_out/bench_qaoa2.json 2> gpurun_out/bench_qaoa2.err
