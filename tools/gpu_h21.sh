cd $GRAFT_REPO_ROOT
PHI_TRACE=1 timeout 300 python tools/probe_blocks.py 3 6 8e-4 > gpurun_out/h21_blocks_c2.out 2>&1
PHI_TRACE=1 timeout 300 python tools/probe_blocks.py 4 7 1.6e-4 > gpurun_out/h21_blocks_c3.out 2>&1
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_determinism.py tests/test_gpu_parity.py -x -q > gpurun_out/h21_pytest.out 2>&1
echo "rc=$?" >> gpurun_out/h21_pytest.out
timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/h21_c2.json 2> gpurun_out/h21_c2.err
timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/h21_c3.json 2> gpurun_out/h21_c3.err
