#!/bin/bash
# Regenerate the round's measurement evidence on a GPU box (run under gpurun):
#   tools/profile_round.sh TAG
# -> gpurun_out/TAG/{bench_c2.json, bench_configs.jsonl, slab_modes.jsonl, launches.csv,
#                    full_c2.ncu-rep, full_c5_raycast.ncu-rep, *.log}
# Each ncu command runs only after the same command exited 0 without ncu.
set -u
tag=${1:-prof}
out=gpurun_out/$tag
mkdir -p $out
# 1. the default bench line (c2, the oracle cpu_baseline, the partitioned path at N = 1)
timeout 1200 python bench.py > $out/bench_c2.json 2> $out/bench_c2.log
echo "bench default rc=$?"
# 2. every config
: > $out/bench_configs.jsonl
for c in 0 1 2 3 4; do
  timeout 900 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline --no-partitioned \
    >> $out/bench_configs.jsonl 2>> $out/bench_configs.log
  echo "bench config $c rc=$?"
done
# 3. the partitioned path's three modes on one rank (c5)
: > $out/slab_modes.jsonl
for mode in segments reduce_scatter fused; do
  timeout 900 python bench.py --slab --config 4 --slab-mode $mode --steps 20 --warmup 3 \
    >> $out/slab_modes.jsonl 2>> $out/slab_modes.log
  echo "slab $mode rc=$?"
done
# 4. launch list of the default command (plain run first)
cmd="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-partitioned --no-l2-probe"
timeout 600 $cmd > /dev/null 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_|FillFunctor" --csv \
    --log-file $out/launches.csv $cmd > $out/launches.log 2>&1
echo "launches rc=$?"
# 5. full sets of one c2 step's kernels (after warm-up)
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_raycast|k_reset_slot|k_finalize_lut|k_endpoint|k_columns|k_negative|k_slope|k_export" \
  -s 16 -c 8 -o $out/full_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-partitioned \
  > $out/full_c2.log 2>&1
echo "full c2 rc=$?"
# 6. the dominant kernel on c5 (largest config)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_raycast -s 2 -c 1 \
  -o $out/full_c5_raycast python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline --no-partitioned \
  > $out/full_c5.log 2>&1
echo "full c5 rc=$?"
# 7. the partitioned path's per-rank cost, P ranks emulated on one GPU (c5)
timeout 1200 python tools/slab_scaling.py 4 > $out/slab_scaling.json 2> $out/slab_scaling.log
echo "slab scaling rc=$?"
