# bench lines and ncu evidence of the final round-2 build (profiles/r02, r02f_*):
# C3 (default) both arms, the multilevel variant c3ml both arms, one full C4
# solve, then the config-3 ncu evidence (launch list, --set full captures of an
# F-relaxation wave, the coarse-march wave and the residual wave).
cd $GRAFT_REPO_ROOT
python bench.py --steps 5 --warmup 3 > gpurun_out/f_c3.json 2> gpurun_out/f_c3.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/f_c3_ref.json 2> gpurun_out/f_c3_ref.err
python bench.py --config c3ml --steps 3 --warmup 3 > gpurun_out/f_c3ml.json 2> gpurun_out/f_c3ml.err
python bench.py --config c3ml --impl reference --steps 2 --warmup 1 > gpurun_out/f_c3ml_ref.json 2> gpurun_out/f_c3ml_ref.err
python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/f_c4.json 2> gpurun_out/f_c4.err
export PHI_WAVE_DEBUG=1
CMD="python tools/probe_breakdown.py c3 1"
$CMD > gpurun_out/f_ncu_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_ncu_launches_c3.csv $CMD > /dev/null 2>&1
for w in 0 4 6; do
  ncu --set full --clock-control none --import-source on -k regex:phi_wave_kernel -s $w -c 1 -o gpurun_out/fw$w $CMD > gpurun_out/f_ncu_w$w.log 2>&1
  python tools/ncu_summary.py full gpurun_out/fw$w.ncu-rep > gpurun_out/f_ncu_w${w}_full.json 2>/dev/null
  ncu -i gpurun_out/fw$w.ncu-rep --page details --csv > gpurun_out/f_ncu_w${w}_details.csv 2>/dev/null
  rm -f gpurun_out/fw$w.ncu-rep
done
