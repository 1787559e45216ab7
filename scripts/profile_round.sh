#!/bin/bash
# Round profiling pass (run under gpurun after `python bench.py` exited 0):
#  1. launch list (gpu__time_duration per launch) of one c2 decode
#  2. ncu --set full of the dominant kernels, one mid-decode launch each
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
CMD="python bench.py --profile-only"
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_c2.csv $CMD > $OUT/launches.log 2>&1
echo "launch list rc $?"
for spec in "gemm_tc_kernel:1300" "att_energy:100" "att_context:100" "seg_scan:200" "pack_rows:1000" \
            "search_step:100" "spec_select:100" "seg_sum:200"; do
  k=${spec%%:*}; skip=${spec##*:}
  ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip $skip -c 1 \
      -o $OUT/full_$k $CMD > $OUT/full_$k.log 2>&1
  echo "full $k rc $?"
done
