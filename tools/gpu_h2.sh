cd $GRAFT_REPO_ROOT
timeout 600 ./tools/spmv_lab 8 > gpurun_out/h2_lab.out 2>&1
# per-block timeline of a single-RHS coarse Phi at the C2 / C3 / C4 shapes (trace build)
PHI_TRACE=1 timeout 300 python tools/probe_blocks.py 3 6 8e-4 > gpurun_out/h2_blocks_c2.out 2>&1
PHI_TRACE=1 timeout 300 python tools/probe_blocks.py 4 7 1.6e-4 > gpurun_out/h2_blocks_c3.out 2>&1
PHI_TRACE=1 timeout 600 python tools/probe_blocks.py 5 8 8e-5 > gpurun_out/h2_blocks_c4.out 2>&1
