#!/bin/bash
timeout 300 python scripts/bench_gemm.py lm_out_240 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 2 -c 1 \
  -o gpurun_out/round2_full_gemm_lm_out python scripts/bench_gemm.py lm_out_240 > gpurun_out/ncu_lmout.log 2>&1
echo "rc $?"
