cd $GRAFT_REPO_ROOT
timeout 600 ./tools/spmv_lab 8 > gpurun_out/h9_lab.out 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/h9_pytest.out 2>&1
echo "pytest rc=$?" >> gpurun_out/h9_pytest.out
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/h9_c3.json 2> gpurun_out/h9_c3.err
