cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_ilut.py -x -v -s --durations=0 > gpurun_out/g7_ilut.out 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 --deselect tests/test_gpu_baseline_parity.py > gpurun_out/g7_gpu.out 2>&1
