cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -s --timeout 600 -p no:cacheprovider > gpurun_out/pytest_multiproc.log 2>&1; echo rc=$? >> gpurun_out/pytest_multiproc.log
QSB_ALL_RANKS_ON_DEVICE0=1 timeout 900 python bench.py --gpus 2 --local-qubits 28 --steps 3 --warmup 3 > gpurun_out/bench_n2_emul.json 2> gpurun_out/bench_n2_emul.err; echo rc=$? >> gpurun_out/bench_n2_emul.err
QSB_ALL_RANKS_ON_DEVICE0=1 timeout 900 python bench.py --gpus 2 --local-qubits 28 --steps 3 --warmup 3 --exchange nccl > gpurun_out/bench_n2_emul_nccl.json 2> gpurun_out/bench_n2_emul_nccl.err; echo rc=$? >> gpurun_out/bench_n2_emul_nccl.err
