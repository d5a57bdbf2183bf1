# bench lines of the final round-2 build (profiles/r02, r02g_*): C3 (default),
# C2, C1, config 5, the multilevel variant c3ml, one full C4 solve.
cd $GRAFT_REPO_ROOT
python bench.py --steps 5 --warmup 3 > gpurun_out/g_c3.json 2> gpurun_out/g_c3.err
python bench.py --config c2 --steps 10 --warmup 3 > gpurun_out/g_c2.json 2> gpurun_out/g_c2.err
python bench.py --config c1 --steps 10 --warmup 3 > gpurun_out/g_c1.json 2> gpurun_out/g_c1.err
python bench.py --config c5 --steps 5 > gpurun_out/g_c5.json 2> gpurun_out/g_c5.err
python bench.py --config c3ml --steps 3 --warmup 3 > gpurun_out/g_c3ml.json 2> gpurun_out/g_c3ml.err
python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/g_c4.json 2> gpurun_out/g_c4.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.out 2>&1
