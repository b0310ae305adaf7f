cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
QSB_DEBUG_TIME=1 timeout 300 python tools/exp/qaoa_step_prof.py > gpurun_out/qaoa_step_prof7.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider -k "factored or optimize or pso or noise" > gpurun_out/pytest_sel7.log 2>&1; echo rc=$? >> gpurun_out/pytest_sel7.log
