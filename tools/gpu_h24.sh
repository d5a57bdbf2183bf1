cd $GRAFT_REPO_ROOT
PHI_CLUSTER=0 PHI_TRACE=1 timeout 300 python tools/probe_point.py 4 7 4e-5 > gpurun_out/h24_point_c3.out 2>&1
PHI_CLUSTER=0 PHI_TRACE=1 timeout 300 python tools/probe_point.py 3 6 1e-4 > gpurun_out/h24_point_c2.out 2>&1
PHI_CLUSTER=0 PHI_TRACE=1 timeout 600 python tools/probe_point.py 5 8 1e-5 > gpurun_out/h24_point_c4.out 2>&1
