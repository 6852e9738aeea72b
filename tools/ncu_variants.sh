#!/bin/bash
# per-kernel mean launch time of a kernel regex for libgvom variants:
# tools/ncu_variants.sh CONFIG REGEX "variants"
c=$1; rx=$2; vars=$3
for v in $vars; do
  if [ "$v" = cur ]; then lib=""; else lib=paper_2109_13176_b200/lib/variants/$v.so; fi
  GVOM_LIBRARY=$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$rx" --csv \
     --log-file gpurun_out/nv_$v.csv python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  echo "NV $v $(python tools/launch_summary.py gpurun_out/nv_$v.csv | sed -n 2,4p | tr '\n' ' ')"
done
