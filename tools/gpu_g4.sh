cd $GRAFT_REPO_ROOT
for a in "3 6 8e-4" "4 7 1.6e-4" "5 8 8e-5"; do
  timeout 300 python tools/probe_blocks.py $a 2>&1 | grep -v "smem plan" >> gpurun_out/g4.out
done
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_parity.py -x -q > gpurun_out/g4_pytest.out 2>&1
timeout 600 python tools/probe_breakdown.py c2 > gpurun_out/g4_c2.out 2> gpurun_out/g4_c2.err
timeout 600 python tools/probe_breakdown.py c3 > gpurun_out/g4_c3.out 2> gpurun_out/g4_c3.err
