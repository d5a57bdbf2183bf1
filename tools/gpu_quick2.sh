#!/bin/bash
# build here first; then: GPU tests, V-cycle probe, C2 bench (no CPU baseline)
mkdir -p gpurun_out
timeout 400 python -u -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 100 python -u tools/probe_vc.py 3 6 0 > gpurun_out/vc.log 2>&1
timeout 300 python bench.py --config ${CFG:-c2} --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench_plain.log 2>&1; echo "rc=$?" >> gpurun_out/bench_plain.log
