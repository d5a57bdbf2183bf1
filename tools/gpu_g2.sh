cd $GRAFT_REPO_ROOT
export PHI_PLAN_DEBUG=1
for a in "3 6 8e-4" "4 7 1.6e-4" "5 8 8e-5"; do
  timeout 300 python tools/probe_blocks.py $a >> gpurun_out/g2.out 2>&1
done
