cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
QSB_DEBUG_TMA=1 QSB_DEBUG_PLAN=1 timeout 300 python tools/exp/qaoa_passes.py factored > gpurun_out/qaoa_plan.txt 2>&1
QSB_NO_TMA=1 timeout 300 python tools/exp/qaoa_passes.py factored >> gpurun_out/qaoa_plan.txt 2>&1
