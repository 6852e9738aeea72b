#!/bin/bash
# ncu launch times + full sets of the integrate kernels on c2 (one step after warm-up)
mkdir -p gpurun_out/pi
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:"k_" --csv \
  --log-file gpurun_out/pi/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-partitioned > gpurun_out/pi/l.log 2>&1
echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_reset_slot|k_finalize_lut|k_endpoint|k_raycast" -s 12 -c 4 -o gpurun_out/pi/integ \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-partitioned > gpurun_out/pi/f.log 2>&1
echo full rc=$?
