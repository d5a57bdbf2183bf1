cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --config c5 --steps 5 > gpurun_out/h20_c5.json 2> gpurun_out/h20_c5.err
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/h20_pytest.out 2>&1
echo "pytest rc=$?" >> gpurun_out/h20_pytest.out
timeout 600 python bench.py --config c2 --steps 5 --warmup 3 > gpurun_out/h20_c2.json 2> gpurun_out/h20_c2.err
timeout 600 python bench.py --config c1 --steps 10 --warmup 3 > gpurun_out/h20_c1.json 2> gpurun_out/h20_c1.err
