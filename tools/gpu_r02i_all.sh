# final check of the committed tree (NVTX ranges, per-solve count assertions in
# test_gpu_fast, bounded reference arm): GPU tier, smoke, both bench arms
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/i_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/i_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/i_smoke.out 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/i_c3_ref.json 2> gpurun_out/i_c3_ref.err
python bench.py --steps 3 --warmup 3 > gpurun_out/i_c3.json 2> gpurun_out/i_c3.err
python bench.py --config c5 --steps 5 > gpurun_out/i_c5.json 2> gpurun_out/i_c5.err
