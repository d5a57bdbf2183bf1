# full GPU tier of the current build + smoke + C2 bench (quick)
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/h1_pytest.out 2>&1
echo "pytest rc=$?" >> gpurun_out/h1_pytest.out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h1_smoke.out 2>&1
timeout 600 python bench.py --config c2 --steps 5 --warmup 3 > gpurun_out/h1_c2.json 2> gpurun_out/h1_c2.err
timeout 600 python bench.py --config c5 --steps 5 > gpurun_out/h1_c5.json 2> gpurun_out/h1_c5.err
