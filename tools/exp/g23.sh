cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --workload cfg1 --steps 20 > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err
timeout 900 python bench.py --workload cfg3 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
timeout 900 python bench.py --workload cfg4 --no-config4-point > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
