#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"seg_scan|seg_sum|row_norm" -s 60 -c 3 \
  -o gpurun_out/round2_full_grows python bench.py --profile-only > gpurun_out/ncu_grows.log 2>&1
echo "capture rc $?"
