cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_comm.py -x -q --durations=10 > gpurun_out/g9_pytest.out 2>&1
