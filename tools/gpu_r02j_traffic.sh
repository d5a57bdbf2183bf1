# DRAM bytes of the serial coarse-march wave of config 3 (launch 4 of the probe) on the final build
cd $GRAFT_REPO_ROOT
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --clock-control none -k regex:phi_wave_kernel -s 4 -c 1 --csv --log-file gpurun_out/j_w4_traffic.csv python tools/probe_breakdown.py c3 1 > gpurun_out/j_w4_traffic.log 2>&1
