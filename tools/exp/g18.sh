cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
for v in prev cur prev cur; do
  if [ $v = cur ]; then L=; else L=scratch/$v/libqsb200.so; fi
  QSB_LIB=$L TAG=$v timeout 120 python tools/exp/pass_times.py >> gpurun_out/ab4.jsonl 2>&1
done
