cd $GRAFT_REPO_ROOT
for a in "3 6 8e-4" "4 7 1.6e-4" "5 8 8e-5"; do
  timeout 300 python tools/probe_blocks.py $a 2>&1 | grep -v "smem plan" | grep -v "^ " >> gpurun_out/g5.out
  PHI_TRACE=0 timeout 300 python tools/probe_blocks.py $a 2>&1 | grep "step wall" >> gpurun_out/g5.out
done
timeout 600 python tools/probe_breakdown.py c2 > gpurun_out/g5_c2.out 2> gpurun_out/g5_c2.err
