#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"seg_scan|seg_sum" -s 40 -c 8 \
  -o gpurun_out/round2_full_grows2 python bench.py --profile-only > gpurun_out/ncu_grows.log 2>&1
echo "capture rc $?"
