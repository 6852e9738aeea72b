timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_gpu_slab.py tests/test_gpu_rolling.py -x -q > gpurun_out/t24.log 2>&1; echo tests rc=$?; grep -E "assert |FAILED|Error" gpurun_out/t24.log | head -5; tail -1 gpurun_out/t24.log
bash tools/ab_env.sh "1 3 4" "- GVOM_NEG_C=1" 30 2>&1 | tee gpurun_out/ab24.log
timeout 600 python tools/slab_rank_stages.py 8 0 4 2>&1 | tail -1
