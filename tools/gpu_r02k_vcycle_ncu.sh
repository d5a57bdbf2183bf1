# ncu --set full of the config-5 V-cycle kernel (p=5; B=64: clusters of 2, B=1: one cluster of 16)
cd $GRAFT_REPO_ROOT
for b in 64 1; do
  python tools/c5_one.py 5 $b 1 > gpurun_out/k_vc_plain_$b.log 2>&1 || exit 1
  timeout 500 ncu --set full --clock-control none -k regex:vcycle_kernel -s 1 -c 1 -o gpurun_out/kvc$b python tools/c5_one.py 5 $b 1 > gpurun_out/k_vc_ncu_$b.log 2>&1
  ncu -i gpurun_out/kvc$b.ncu-rep --page raw --csv > gpurun_out/k_vc_${b}_raw.csv 2>/dev/null
  ncu -i gpurun_out/kvc$b.ncu-rep --page details --csv > gpurun_out/k_vc_${b}_details.csv 2>/dev/null
  rm -f gpurun_out/kvc$b.ncu-rep
done
