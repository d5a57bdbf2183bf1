cd $GRAFT_REPO_ROOT
export PHI_WAVE_DEBUG=1
CUDA_MODULE_LOADING=EAGER timeout 600 python tools/probe_breakdown.py c3 2 > gpurun_out/g19_c3_eager.out 2>&1
timeout 600 python tools/probe_breakdown.py c3 2 > gpurun_out/g19_c3_lazy.out 2>&1
