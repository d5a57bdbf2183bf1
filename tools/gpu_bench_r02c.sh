# bench lines of the current build (profiles/r02): C3 (default) both arms,
# the multilevel variant c3ml both arms, config 5, one full C4 solve.
cd $GRAFT_REPO_ROOT
python bench.py --steps 5 --warmup 3 > gpurun_out/b_c3.json 2> gpurun_out/b_c3.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/b_c3_ref.json 2> gpurun_out/b_c3_ref.err
python bench.py --config c3ml --steps 3 --warmup 3 > gpurun_out/b_c3ml.json 2> gpurun_out/b_c3ml.err
python bench.py --config c3ml --impl reference --steps 2 --warmup 1 > gpurun_out/b_c3ml_ref.json 2> gpurun_out/b_c3ml_ref.err
python bench.py --config c5 --steps 5 > gpurun_out/b_c5.json 2> gpurun_out/b_c5.err
python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err
