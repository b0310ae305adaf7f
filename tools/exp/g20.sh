cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU="ncu --set full --import-source on --clock-control none"
M=30 REPS=1 timeout 900 $NCU -k regex:k_fact --launch-skip 9 --launch-count 3 -o gpurun_out/r02c_fact python tools/exp/pass_times.py > gpurun_out/ncu_fact.log 2>&1
ncu -i gpurun_out/r02c_fact.ncu-rep --page raw --csv > gpurun_out/r02c_fact.raw.csv 2>/dev/null
rm -f gpurun_out/r02c_fact.ncu-rep
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02c.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-per-target --no-exact-compare --no-config4-point > gpurun_out/ncu_launch.log 2>&1
