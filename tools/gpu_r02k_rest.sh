# the remaining bench lines of the final build (profiles/r02, r02k_*): C1, config 5, one full C4 solve
cd $GRAFT_REPO_ROOT
python bench.py --config c1 --steps 10 --warmup 3 > gpurun_out/k_c1.json 2> gpurun_out/k_c1.err
python bench.py --config c5 --steps 5 > gpurun_out/k_c5.json 2> gpurun_out/k_c5.err
python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/k_c4.json 2> gpurun_out/k_c4.err
