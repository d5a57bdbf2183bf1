cd $GRAFT_REPO_ROOT
timeout 600 ./tools/spmv_lab 8 > gpurun_out/h11_lab.out 2>&1
