#!/bin/bash
mkdir -p gpurun_out/pc
for k in 0 1000 64; do
  GVOM_RAY_CHUNK=$k timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('chunk=$k', 'step_ms=%.4f'%d['ms_per_step'], 'ray_ms=%.4f'%d['roofline']['launch_ms'], 'integ=%.4f'%d['integrate']['ms_per_frame'], 'maps=%.4f'%d['compute_maps_ms']); print(json.dumps(d['roofline']['l2_red']))"
done
GVOM_SLOPE_PERCELL=1 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('slope percell', 'step_ms=%.4f'%d['ms_per_step'], 'maps=%.4f'%d['compute_maps_ms'], d['stages_ms_per_step'])"
GVOM_RAY_CHUNK=0 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('slope compact', 'step_ms=%.4f'%d['ms_per_step'], 'maps=%.4f'%d['compute_maps_ms'], d['stages_ms_per_step'])"
GVOM_RAY_CHUNK=64 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_raycast_q -s 3 -c 1 -o gpurun_out/pc/chunk64 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/pc/ncu64.log 2>&1
echo ncu rc=$?
GVOM_RAY_CHUNK=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_raycast|k_finalize_frame|k_columns|k_negative_tb|k_slope_c|k_neg_decide" -s 18 -c 7 -o gpurun_out/pc/step0 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/pc/ncu0.log 2>&1
echo ncu0 rc=$?
