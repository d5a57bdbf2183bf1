mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -15
python tools/probe_units.py 2>&1 | tail -3
python tools/probe_waves.py c2 2>&1 | grep -E "wave [0-9] |wave 1[0-2] |^\(" 
