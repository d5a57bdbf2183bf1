cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt
nproc >> gpurun_out/g1_smi.txt
timeout 600 python tools/probe_breakdown.py c3 > gpurun_out/g1_c3.out 2> gpurun_out/g1_c3.err
timeout 900 python tools/probe_breakdown.py c4 1 > gpurun_out/g1_c4.out 2> gpurun_out/g1_c4.err
