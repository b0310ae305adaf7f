cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 tools/exp/tma_tilecopy > gpurun_out/tma_tilecopy4.txt 2>&1
