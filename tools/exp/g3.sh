cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 tools/exp/tma_tilecopy > gpurun_out/tma_tilecopy.txt 2>&1
timeout 300 python tools/exp/sweep_order.py > gpurun_out/sweep_order.jsonl 2>&1
QSB_TMA_PF=0 timeout 300 python tools/exp/sweep_order.py > gpurun_out/sweep_order_pf0.jsonl 2>&1
timeout 600 python bench.py --workload qaoa > gpurun_out/bench_qaoa.json 2> gpurun_out/bench_qaoa.err
