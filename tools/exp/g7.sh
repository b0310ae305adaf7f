cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/ab_sweep.jsonl gpurun_out/ab_qaoa.txt
for v in cur head cur; do
  if [ $v = cur ]; then L=; else L=scratch/$v/libqsb200.so; fi
  QSB_LIB=$L TAG=$v timeout 300 python tools/exp/pass_times.py >> gpurun_out/ab_sweep.jsonl 2>&1
  QSB_LIB=$L timeout 300 python tools/exp/qaoa_passes.py factored 2>&1 | grep total | sed "s/^/$v /" >> gpurun_out/ab_qaoa.txt
done
QSB_TMA_PF=1 timeout 300 python tools/exp/qaoa_passes.py factored 2>&1 | grep total | sed "s/^/cur_pf1 /" >> gpurun_out/ab_qaoa.txt
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --workload qaoa > gpurun_out/bench_qaoa.json 2> gpurun_out/bench_qaoa.err
timeout 600 python bench.py --workload noise > gpurun_out/bench_noise.json 2> gpurun_out/bench_noise.err
