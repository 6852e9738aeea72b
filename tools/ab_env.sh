#!/bin/bash
# A/B timing of environment switches: tools/ab_env.sh "cfgs" "VAR=a VAR=b ..." [steps]
# ("-" = no override)
cfgs=${1:-"1"}; vars=${2:-"-"}; steps=${3:-50}
for rep in 1 2; do
for c in $cfgs; do for v in $vars; do
  if [ "$v" = "-" ]; then envs=""; else envs="${v//,/ }"; fi
  env $envs timeout 600 python bench.py --config $c --steps $steps --warmup 5 --no-cpu-baseline --no-partitioned --no-l2-probe 2>/dev/null | tail -1 | \
    python -c "import json,sys;d=json.loads(sys.stdin.read());st=d['stages_ms_per_step'];print('AB', '$v', d['config']['workload'][:3], 'step_ms=%.4f'%d['ms_per_step'], 'ray_ms=%.4f'%d['roofline']['launch_ms'], 'integ_ms=%.4f'%d['integrate']['ms_per_frame'], 'maps_ms=%.4f'%d['compute_maps_ms'], 'stages', {k: round(v*1000,1) for k,v in st.items()})"
done; done; done
