cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/exp/qaoa_step_prof.py > gpurun_out/qaoa_step_prof6.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider -k "optimize or pso or cli or noise or dropin or pool or ref" > gpurun_out/pytest_sel6.log 2>&1; echo rc=$? >> gpurun_out/pytest_sel6.log
timeout 600 python bench.py --workload qaoa > gpurun_out/bench_qaoa6.json 2> gpurun_out/bench_qaoa6.err
