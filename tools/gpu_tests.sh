#!/bin/bash
# run the GPU test suite; print a one-line summary (and failures) for gpurun's tail
timeout ${1:-900} python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
rc=$?
grep -E "Error|assert |FAILED" gpurun_out/gpu_tests.log | head -8
echo "GPU-TESTS rc=$rc $(tail -1 gpurun_out/gpu_tests.log)"
