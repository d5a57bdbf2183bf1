cd $GRAFT_REPO_ROOT
./tools/ldsrate_probe > gpurun_out/h4_ldsrate.out 2>&1
timeout 900 ./tools/spmv_lab 8 > gpurun_out/h4_lab.out 2>&1
