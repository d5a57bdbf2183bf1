# validation of the lower-triangle block inverses as the default build: GPU tier,
# smoke, bench lines (C3 default, C2, c3ml), and an ncu --set full capture of the
# serial coarse-march wave of config 3 (launch 4 of the probe) for its DRAM bytes
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/j_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/j_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/j_smoke.out 2>&1
python bench.py --steps 3 --warmup 3 > gpurun_out/j_c3.json 2> gpurun_out/j_c3.err
python bench.py --config c2 --steps 10 --warmup 3 > gpurun_out/j_c2.json 2> gpurun_out/j_c2.err
python bench.py --config c3ml --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/j_c3ml.json 2> gpurun_out/j_c3ml.err
CMD="python tools/probe_breakdown.py c3 1"
timeout 900 ncu --set full --clock-control none -k regex:phi_wave_kernel -s 4 -c 1 -o gpurun_out/jw4 $CMD > gpurun_out/j_ncu_w4.log 2>&1
ncu -i gpurun_out/jw4.ncu-rep --page raw --csv > gpurun_out/j_ncu_w4_raw.csv 2>/dev/null
ncu -i gpurun_out/jw4.ncu-rep --page details --csv > gpurun_out/j_ncu_w4_details.csv 2>/dev/null
rm -f gpurun_out/jw4.ncu-rep
