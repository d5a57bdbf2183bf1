cd $GRAFT_REPO_ROOT
PHI_TRACE=1 timeout 300 python tools/probe_blocks.py 3 6 8e-4 > gpurun_out/h23_blocks_c2.out 2>&1
PHI_TRACE=1 timeout 300 python tools/probe_blocks.py 4 7 1.6e-4 > gpurun_out/h23_blocks_c3.out 2>&1
PHI_TRACE=1 timeout 600 python tools/probe_blocks.py 5 8 8e-5 > gpurun_out/h23_blocks_c4.out 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/h23_pytest.out 2>&1
echo "pytest rc=$?" >> gpurun_out/h23_pytest.out
timeout 600 python bench.py --config c2 --steps 5 --warmup 3 > gpurun_out/h23_c2.json 2> gpurun_out/h23_c2.err
timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/h23_c3.json 2> gpurun_out/h23_c3.err
