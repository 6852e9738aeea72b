python tools/scratch/probe_mc.py 2>&1 | tail -40
