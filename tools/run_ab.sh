timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr 127.0.0.1 --master-port 29733 tools/slab_step_parts.py 2>/dev/null | tail -1
for r in 1 2; do timeout 600 python bench.py --slab --config 4 --slab-mode segments --steps 20 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('SLAB', d['ms_per_step'])"; done
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random.py tests/test_gpu_step.py tests/test_gpu_rolling.py tests/test_gpu_shapes.py -x -q > gpurun_out/t29.log 2>&1; echo tests rc=$?; grep -E "assert |FAILED|Error" gpurun_out/t29.log | head -5; tail -1 gpurun_out/t29.log
bash tools/ab_env.sh "1 2 3" "- GVOM_EP_FUSED=0" 50 2>&1 | tee gpurun_out/ab29.log
