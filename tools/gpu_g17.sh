cd $GRAFT_REPO_ROOT
export PHI_WAVE_DEBUG=1
for o in 0 1; do
  PHI_OVERLAP=$o timeout 600 python tools/probe_breakdown.py c3 1 > gpurun_out/g17_c3_o$o.out 2>&1
  PHI_OVERLAP=$o timeout 600 python tools/probe_breakdown.py c2 1 > gpurun_out/g17_c2_o$o.out 2>&1
done
