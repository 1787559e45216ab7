#!/bin/bash
# round-2 GPU job g: stats fix + remaining c4 drift source
mkdir -p gpurun_out
timeout 300 python scripts/stats_debug.py > gpurun_out/stats_debug.log 2>&1; tail -4 gpurun_out/stats_debug.log
timeout 300 python -m pytest tests/test_gpu_gemm.py -m gpu -q > gpurun_out/pytest_gemm.log 2>&1; tail -1 gpurun_out/pytest_gemm.log
for c in c5 c4; do timeout 300 python scripts/parity_dump.py $c g > /dev/null 2>&1; done
FB_KCB_LM=1 timeout 300 python scripts/parity_dump.py c4 glm > /dev/null 2>&1
timeout 600 python scripts/step_error.py c4 1822 > gpurun_out/step_error_c4g.log 2>&1; tail -9 gpurun_out/step_error_c4g.log
