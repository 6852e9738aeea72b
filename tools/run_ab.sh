timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random.py tests/test_gpu_step.py tests/test_gpu_variants.py tests/test_gpu_slab.py -x -q > gpurun_out/t18.log 2>&1; echo tests rc=$?; grep -E "assert |FAILED|Error" gpurun_out/t18.log | head -5; tail -1 gpurun_out/t18.log
bash tools/ab_env.sh "1 2 3" "- GVOM_FIN_FUSED=1" 50 2>&1 | tee gpurun_out/ab18.log
