cd $GRAFT_REPO_ROOT
PHI_TRACE=1 timeout 300 python tools/probe_blocks.py 3 6 8e-4 > gpurun_out/h8_blocks_c2.out 2>&1
PHI_TRACE=1 timeout 300 python tools/probe_blocks.py 4 7 1.6e-4 > gpurun_out/h8_blocks_c3.out 2>&1
timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/h8_c2.json 2> gpurun_out/h8_c2.err
PHI_VARIANT=ns3 timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/h8_c2_ns3.json 2> gpurun_out/h8_c2_ns3.err
PHI_OVERLAP=1 timeout 600 python tools/probe_breakdown.py c3 2 2>/dev/null | tail -1 > gpurun_out/h8_c3_ns2.out
PHI_VARIANT=ns3 PHI_OVERLAP=1 timeout 600 python tools/probe_breakdown.py c3 2 2>/dev/null | tail -1 > gpurun_out/h8_c3_ns3.out
