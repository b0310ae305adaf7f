cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
FUSE=exact TAG=exact_lean timeout 300 python tools/exp/pass_times.py > gpurun_out/pt_exact.jsonl 2>&1
QSB_NO_EXACT_LEAN=1 FUSE=exact TAG=exact_ktile timeout 300 python tools/exp/pass_times.py >> gpurun_out/pt_exact.jsonl 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
