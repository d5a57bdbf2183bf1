cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_overlap.py tests/test_gpu_fast.py tests/test_gpu_parity.py tests/test_gpu_determinism.py tests/test_gpu_comm.py tests/test_gpu_timeshard.py tests/test_gpu_baseline_parity.py -x -q -k "not config4_shape_exact and not config5" > gpurun_out/g16_pytest.out 2>&1
for o in 0 1; do
  PHI_OVERLAP=$o timeout 300 python tools/probe_breakdown.py c2 2>/dev/null | tail -1 > gpurun_out/g16_c2_o$o.out
  PHI_OVERLAP=$o timeout 600 python tools/probe_breakdown.py c3 2>/dev/null | tail -1 > gpurun_out/g16_c3_o$o.out
done
