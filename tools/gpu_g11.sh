cd $GRAFT_REPO_ROOT
export PHI_WAVE_DEBUG=1
python tools/probe_breakdown.py c3 1 > gpurun_out/g11_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g11_launches_c3.csv \
    python tools/probe_breakdown.py c3 1 > gpurun_out/g11_ncu_launches.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:phi_wave_kernel -s 0 -c 7 \
    -o gpurun_out/g11_c3_waves python tools/probe_breakdown.py c3 1 > gpurun_out/g11_ncu_full.log 2>&1
echo "rc=$?" >> gpurun_out/g11_ncu_full.log
