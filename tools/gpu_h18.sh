cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_baseline_parity.py -x -q -k "config5 or config4_multilevel" > gpurun_out/h18_pytest.out 2>&1
echo "rc=$?" >> gpurun_out/h18_pytest.out
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_determinism.py tests/test_gpu_comm.py -x -q > gpurun_out/h18_pytest2.out 2>&1
echo "rc=$?" >> gpurun_out/h18_pytest2.out
timeout 900 python bench.py --config c5 --steps 5 > gpurun_out/h18_c5.json 2> gpurun_out/h18_c5.err
timeout 900 python bench.py --config c3ml --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/h18_c3ml.json 2> gpurun_out/h18_c3ml.err
