cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_determinism.py -x -q > gpurun_out/h3_pytest_fast.out 2>&1
echo "rc=$?" >> gpurun_out/h3_pytest_fast.out
PHI_TRACE=1 timeout 300 python tools/probe_blocks.py 3 6 8e-4 > gpurun_out/h3_blocks_c2.out 2>&1
PHI_TRACE=1 timeout 300 python tools/probe_blocks.py 4 7 1.6e-4 > gpurun_out/h3_blocks_c3.out 2>&1
PHI_TRACE=1 timeout 600 python tools/probe_blocks.py 5 8 8e-5 > gpurun_out/h3_blocks_c4.out 2>&1
timeout 600 python bench.py --config c2 --steps 3 --warmup 3 > gpurun_out/h3_c2.json 2> gpurun_out/h3_c2.err
timeout 900 python -m pytest tests/test_gpu_baseline_parity.py -x -q -k "config2 or config3_two or config5" > gpurun_out/h3_pytest_parity.out 2>&1
echo "rc=$?" >> gpurun_out/h3_pytest_parity.out
