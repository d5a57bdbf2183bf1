#!/bin/bash
# One GPU-box pass: GPU parity tests, smoke, a bench line, the ncu launch list
# and one full ncu capture of the dominant kernel (each ncu pass only after the
# same command exited 0 without ncu).  Outputs land in gpurun_out/.
set -u
mkdir -p gpurun_out
TAG=${TAG:-r01}
CFG=${CFG:-c2}
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench_plain.log 2>&1
rc=$?
echo "bench rc=$rc" >> gpurun_out/bench_plain.log
if [ $rc -eq 0 ] && [ "${NCU:-1}" = 1 ]; then
  ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv \
      --log-file gpurun_out/launches_$TAG.csv \
      python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:phi_wave_kernel --launch-skip ${SKIP:-6} -c 1 \
      -o gpurun_out/phi_wave_$TAG -f \
      python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
fi
