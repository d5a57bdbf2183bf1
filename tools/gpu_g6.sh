cd $GRAFT_REPO_ROOT
nproc > gpurun_out/g6_nproc.txt
timeout 1700 python -m pytest tests/test_gpu_baseline_parity.py -x -v -s --durations=0 > gpurun_out/g6_pytest.out 2>&1
