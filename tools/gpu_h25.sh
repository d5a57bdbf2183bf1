cd $GRAFT_REPO_ROOT
PHI_CLUSTER=0 PHI_TRACE=1 timeout 300 python tools/probe_point.py 4 7 4e-5 > gpurun_out/h25_point_c3.out 2>&1
PHI_CLUSTER=0 PHI_TRACE=1 timeout 300 python tools/probe_point.py 3 6 1e-4 > gpurun_out/h25_point_c2.out 2>&1
PHI_CLUSTER=0 PHI_TRACE=1 timeout 600 python tools/probe_point.py 5 8 1e-5 > gpurun_out/h25_point_c4.out 2>&1
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_determinism.py -x -q > gpurun_out/h25_pytest.out 2>&1
echo "rc=$?" >> gpurun_out/h25_pytest.out
timeout 900 python bench.py --config c3ml --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/h25_c3ml.json 2> gpurun_out/h25_c3ml.err
timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/h25_c3.json 2> gpurun_out/h25_c3.err
