cd $GRAFT_REPO_ROOT
export PHI_WAVE_DEBUG=1 PHI_OVERLAP_DEBUG=1
timeout 600 python tools/probe_breakdown.py c3 1 > gpurun_out/g18_c3.out 2>&1
