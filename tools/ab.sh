#!/bin/bash
# A/B timing of libgvom variants: tools/ab.sh "cfgs" "variants" [steps]
# variants are names under paper_2109_13176_b200/lib/variants ("cur" = lib/libgvom.so)
cfgs=${1:-"1 4"}; vars=${2:-"cur"}; steps=${3:-20}
for rep in 1 2; do
for c in $cfgs; do for v in $vars; do
  if [ "$v" = cur ]; then lib=""; else lib=paper_2109_13176_b200/lib/variants/$v.so; fi
  GVOM_LIBRARY=$lib timeout 600 python bench.py --config $c --steps $steps --warmup 5 --no-cpu-baseline --no-partitioned --no-l2-probe 2>/dev/null | tail -1 | \
    python -c "import json,sys;d=json.loads(sys.stdin.read());print('AB', '$v', d['config']['workload'][:3], 'step_ms=%.4f'%d['ms_per_step'], 'ray_ms=%.4f'%d['roofline']['launch_ms'], 'frac=%.3f'%d['roofline']['frac'], 'e2e=%.0f'%(d['e2e']['value']/1e6))"
done; done; done
