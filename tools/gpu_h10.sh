cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_fast.py -x -q -k spmm > gpurun_out/h10_pytest.out 2>&1
echo "rc=$?" >> gpurun_out/h10_pytest.out
timeout 900 python bench.py --config c5 --steps 5 > gpurun_out/h10_c5.json 2> gpurun_out/h10_c5.err
# ncu: the p=5 SpMV and the p=5 B=64 / B=16 SpMM (after the plain runs exited 0)
for pb in "5 1" "5 64" "5 16" "2 1"; do
  set -- $pb
  python tools/c5_one.py $1 $2 > gpurun_out/h10_one_$1_$2.log 2>&1 || continue
  ncu --set full --clock-control none --import-source on -k regex:sp.._tma_kernel -s 1 -c 1 -o gpurun_out/k_$1_$2 python tools/c5_one.py $1 $2 > gpurun_out/h10_ncu_$1_$2.log 2>&1
  python tools/ncu_summary.py full gpurun_out/k_$1_$2.ncu-rep > gpurun_out/h10_full_$1_$2.json 2>/dev/null
  ncu -i gpurun_out/k_$1_$2.ncu-rep --page details --csv > gpurun_out/h10_details_$1_$2.csv 2>/dev/null
  rm -f gpurun_out/k_$1_$2.ncu-rep
done
