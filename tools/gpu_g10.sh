cd $GRAFT_REPO_ROOT
S=/usr/local/cuda/bin/compute-sanitizer
timeout 600 python -m pytest tests/test_gpu_binding.py tests/test_gpu_fast.py tests/test_gpu_parity.py -x -q > gpurun_out/g10_pytest.out 2>&1
timeout 300 python tools/probe_breakdown.py c2 > gpurun_out/g10_c2.out 2>&1
timeout 900 $S --tool racecheck --racecheck-report analysis python tools/sanitize_case.py > gpurun_out/g10_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/g10_racecheck.log
timeout 900 $S --tool synccheck python tools/sanitize_case.py > gpurun_out/g10_synccheck.log 2>&1; echo "rc=$?" >> gpurun_out/g10_synccheck.log
timeout 900 $S --tool memcheck python tools/sanitize_case.py window > gpurun_out/g10_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/g10_memcheck.log
