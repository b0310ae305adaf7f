cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/ab_pool.txt
for v in cur nocut sharedt both cur; do
  if [ $v = cur ]; then L=; else L=scratch/$v/libqsb200.so; fi
  QSB_LIB=$L timeout 300 python tools/exp/qaoa_passes.py factored 2>&1 | grep total | sed "s/^/$v /" >> gpurun_out/ab_pool.txt
done
