cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_fast.py -x -q -k "building or config3_4" > gpurun_out/g15_pytest.out 2>&1
for a in "3 6 8e-4" "4 7 1.6e-4" "5 8 8e-5"; do
  timeout 300 python tools/probe_blocks.py $a 2>&1 | grep -v "smem plan" | grep -v "^  [0-9]" >> gpurun_out/g15.out
  PHI_TRACE=0 timeout 300 python tools/probe_blocks.py $a 2>&1 | grep "step wall" >> gpurun_out/g15.out
done
timeout 300 python tools/probe_breakdown.py c2 > gpurun_out/g15_c2.out 2>/dev/null
timeout 600 python tools/probe_breakdown.py c3 > gpurun_out/g15_c3.out 2>/dev/null
