cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python tools/exp/pass_times.py > gpurun_out/pt_pair2.jsonl 2>&1
NCU="ncu --set full --import-source on --clock-control none"
M=30 REPS=1 timeout 900 $NCU -k regex:k_fact --launch-skip 10 --launch-count 2 -o gpurun_out/pair_p23 python tools/exp/pass_times.py > gpurun_out/ncu_pair.log 2>&1
ncu -i gpurun_out/pair_p23.ncu-rep --page raw --csv > gpurun_out/pair_p23.raw.csv 2>/dev/null
ncu -i gpurun_out/pair_p23.ncu-rep --page source --csv --print-source sass > gpurun_out/pair_p23.source.csv 2>/dev/null
gzip -f gpurun_out/pair_p23.source.csv; rm -f gpurun_out/pair_p23.ncu-rep
