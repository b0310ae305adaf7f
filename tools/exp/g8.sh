cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU="ncu --set full --import-source on --clock-control none"
for v in head cur; do
  if [ $v = cur ]; then L=; else L=scratch/$v/libqsb200.so; fi
  QSB_LIB=$L M=30 REPS=1 timeout 600 $NCU -k regex:k_fact --launch-skip 10 --launch-count 1 -o gpurun_out/p2_$v python tools/exp/pass_times.py > gpurun_out/ncu_p2_$v.log 2>&1
  ncu -i gpurun_out/p2_$v.ncu-rep --page raw --csv > gpurun_out/p2_$v.raw.csv 2>/dev/null
  ncu -i gpurun_out/p2_$v.ncu-rep --page source --csv --print-source sass > gpurun_out/p2_$v.source.csv 2>/dev/null
  gzip -f gpurun_out/p2_$v.source.csv; rm -f gpurun_out/p2_$v.ncu-rep
done
for pf in 0 1; do QSB_TMA_PF=$pf TAG=pf$pf timeout 300 python tools/exp/pass_times.py >> gpurun_out/ab_sweep_pf.jsonl 2>&1; done
