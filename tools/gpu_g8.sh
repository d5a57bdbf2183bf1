cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_timeshard.py tests/test_gpu_baseline_parity.py -x -q -k "timeshard or multilevel or fcycle" --durations=10 > gpurun_out/g8_pytest.out 2>&1
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/g8_bench_c3.out 2> gpurun_out/g8_bench_c3.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/g8_ref_c3.out 2> gpurun_out/g8_ref_c3.err
