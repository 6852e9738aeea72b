#!/bin/bash
# Regenerate the round's measurement evidence on a GPU box (run under gpurun):
#   tools/profile_round.sh TAG
# -> gpurun_out/TAG/{bench_c2.json, bench_configs.jsonl, launches.csv,
#                    full_c2.ncu-rep, full_c5_raycast.ncu-rep, *.log}
# Each ncu command runs only after the same command exited 0 without ncu.
set -u
tag=${1:-prof}
out=gpurun_out/$tag
mkdir -p $out
# 1. the default bench line (c2, with the oracle cpu_baseline) and every config
timeout 900 python bench.py > $out/bench_c2.json 2> $out/bench_c2.log
echo "bench default rc=$?"
: > $out/bench_configs.jsonl
for c in 0 1 2 3 4; do
  timeout 900 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline \
    >> $out/bench_configs.jsonl 2>> $out/bench_configs.log
  echo "bench config $c rc=$?"
done
# 2. launch list of the default command (plain run first)
cmd="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
timeout 600 $cmd > /dev/null 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_|FillFunctor" --csv \
    --log-file $out/launches.csv $cmd > $out/launches.log 2>&1
echo "launches rc=$?"
# 3. full sets of the step's kernels on c2 (one launch each, after warm-up)
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_raycast|k_finalize_tiles|k_endpoint|k_columns|k_negative|k_slope|k_zero3|k_export|k_neg_decide" \
  -s 18 -c 9 -o $out/full_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  > $out/full_c2.log 2>&1
echo "full c2 rc=$?"
# 4. the dominant kernel on c5 (largest config)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_raycast -s 2 -c 1 \
  -o $out/full_c5_raycast python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline \
  > $out/full_c5.log 2>&1
echo "full c5 rc=$?"
