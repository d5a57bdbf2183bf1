# round-2 final validation of the rebuilt library (own-formulation host setup,
# cluster IC projection): the new projection test first, then the whole GPU
# tier, then the default bench line and C2 (profiles/r02, r02h_*)
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_baseline_parity.py -k initial_projection -x -q > gpurun_out/h_proj.log 2>&1; echo "rc=$?" >> gpurun_out/h_proj.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/h_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/h_pytest.log
python bench.py --steps 3 --warmup 3 > gpurun_out/h_c3.json 2> gpurun_out/h_c3.err
python bench.py --config c2 --steps 10 --warmup 3 > gpurun_out/h_c2.json 2> gpurun_out/h_c2.err
PHI_WAVE_DEBUG=1 python tools/probe_breakdown.py c3 1 > gpurun_out/h_breakdown_c3.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/h_ncu_launches_c3.csv python tools/probe_breakdown.py c3 1 > /dev/null 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h_smoke.out 2>&1
