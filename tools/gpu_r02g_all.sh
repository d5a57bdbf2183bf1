# final round-2 validation: GPU test tier, then the bench lines (profiles/r02, r02g_*)
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g_pytest.log
bash tools/gpu_bench_r02g.sh
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/g_c3_ref.json 2> gpurun_out/g_c3_ref.err
