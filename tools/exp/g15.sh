cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python tools/exp/pass_times.py > gpurun_out/pt_pair.jsonl 2>&1
QSB_NO_PAIR=1 TAG=nopair timeout 120 python tools/exp/pass_times.py >> gpurun_out/pt_pair.jsonl 2>&1
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider -k "factored or headline or smoke" > gpurun_out/pytest_pair.log 2>&1; echo rc=$? >> gpurun_out/pytest_pair.log
