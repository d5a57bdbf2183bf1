cd $GRAFT_REPO_ROOT
for o in 0 1; do
  PHI_OVERLAP=$o timeout 300 python tools/probe_breakdown.py c2 2>/dev/null | tail -1 > gpurun_out/g20_c2_o$o.out
  PHI_OVERLAP=$o timeout 600 python tools/probe_breakdown.py c3 2>/dev/null | tail -1 > gpurun_out/g20_c3_o$o.out
done
timeout 600 python -m pytest tests/test_gpu_overlap.py -q -x > gpurun_out/g20_pytest.out 2>&1
