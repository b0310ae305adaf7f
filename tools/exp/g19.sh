cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/ab5.jsonl
for v in prev cur prev cur; do
  if [ $v = cur ]; then L=; else L=scratch/$v/libqsb200.so; fi
  QSB_LIB=$L TAG=$v timeout 120 python tools/exp/pass_times.py >> gpurun_out/ab5.jsonl 2>&1
done
