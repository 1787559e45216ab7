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
# name:skip:count -- the GEMM and pack captures take one whole decode step's
# launches (13 GEMMs, ~8 packs at c2) so every shape of the step is covered
for spec in "gemm_tc_kernel:1300:13" "att_energy:100:1" "att_context:100:1" "seg_scan:200:2" \
            "pack_rows:1000:8" "search_step:100:1" "spec_select:100:1" "seg_sum:200:2"; do
  k=${spec%%:*}; rest=${spec#*:}; skip=${rest%%:*}; cnt=${rest##*:}
  ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip $skip -c $cnt \
      -o $OUT/full_$k $CMD > $OUT/full_$k.log 2>&1
  echo "full $k rc $?"
done
