#!/bin/bash
# one gpurun call: plain QAOA/noise bench lines, then ncu --set full captures of
# the factored sweep (k_fact_tma), the exact sweep (k_tile) and the pool passes
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
R=${ROUND:-r02b}
NCU="ncu --set full --import-source on --clock-control none"
timeout 600 python bench.py --workload qaoa > gpurun_out/bench_qaoa.json 2> gpurun_out/bench_qaoa.err
timeout 600 python bench.py --workload noise > gpurun_out/bench_noise.json 2> gpurun_out/bench_noise.err
M=30 REPS=1 timeout 900 $NCU -k regex:k_fact --launch-skip 9 --launch-count 3 -o gpurun_out/${R}_fact python tools/exp/pass_times.py > gpurun_out/ncu_fact.log 2>&1
M=30 REPS=1 FUSE=exact timeout 900 $NCU -k regex:k_tile --launch-skip 9 --launch-count 3 -o gpurun_out/${R}_tile python tools/exp/pass_times.py > gpurun_out/ncu_tile.log 2>&1
timeout 900 $NCU -k regex:"k_fact|k_tile" --launch-skip 18 --launch-count 6 -o gpurun_out/${R}_qaoa python bench.py --workload qaoa --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_qaoa.log 2>&1
timeout 900 $NCU -k regex:"k_fact|k_tile" --launch-skip 18 --launch-count 6 -o gpurun_out/${R}_noise python bench.py --workload noise --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_noise.log 2>&1
ls -la gpurun_out
