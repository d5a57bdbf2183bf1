# ncu evidence for config 3 (profiles/r02): the launch list of one initialize()
# + MGRIT cycle, and --set full captures of an F-relaxation wave (launch 0),
# the serial coarse-march wave (launch 4) and the residual wave (launch 6).
# Reports are reduced to CSV on the box (gpurun_out is capped at 64 MiB).
cd $GRAFT_REPO_ROOT
export PHI_WAVE_DEBUG=1
CMD="python tools/probe_breakdown.py c3 1"
$CMD > gpurun_out/ncu_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_launches_c3.csv $CMD > /dev/null 2>&1
for w in 0 4 6; do
  ncu --set full --clock-control none -k regex:phi_wave_kernel -s $w -c 1 -o gpurun_out/w$w $CMD > gpurun_out/ncu_w$w.log 2>&1
  ncu -i gpurun_out/w$w.ncu-rep --page raw --csv > gpurun_out/ncu_w${w}_raw.csv 2>/dev/null
  ncu -i gpurun_out/w$w.ncu-rep --page details --csv > gpurun_out/ncu_w${w}_details.csv 2>/dev/null
  rm -f gpurun_out/w$w.ncu-rep
done
ls -la gpurun_out/ > gpurun_out/ncu_ls.txt
