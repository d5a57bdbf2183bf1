cd $GRAFT_REPO_ROOT
export PHI_PLAN_DEBUG=1
for a in "4 7 1.6e-4" "5 8 8e-5"; do
  PHI_TRACE=0 timeout 300 python tools/probe_step.py $a > gpurun_out/g3_step_$(echo $a|tr ' ' _).out 2>&1
  timeout 300 python tools/probe_blocks.py $a 2>&1 | grep -v "smem plan" >> gpurun_out/g3.out
done
timeout 900 python -m pytest tests/test_gpu_fast.py -x -q -k "config3_4 or building or solve_iter" > gpurun_out/g3_pytest.out 2>&1
