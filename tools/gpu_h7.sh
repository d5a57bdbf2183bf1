cd $GRAFT_REPO_ROOT
PHI_TRACE=1 timeout 300 python tools/probe_blocks.py 3 6 8e-4 > gpurun_out/h7_blocks_c2.out 2>&1
PHI_TRACE=1 timeout 300 python tools/probe_blocks.py 4 7 1.6e-4 > gpurun_out/h7_blocks_c3.out 2>&1
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_determinism.py -x -q > gpurun_out/h7_pytest_fast.out 2>&1
echo "rc=$?" >> gpurun_out/h7_pytest_fast.out
timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/h7_c2.json 2> gpurun_out/h7_c2.err
