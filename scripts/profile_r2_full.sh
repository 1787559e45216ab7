#!/bin/bash
# Round-2 profiling at HEAD: launch list of one c2 decode, then `--set full`
# captures of the tcgen05 GEMM (acoustic LSTM shape) and of the look-ahead,
# selection, context and g-row kernels inside a decode (one launch each).
set -u
OUT=gpurun_out/prof3
mkdir -p $OUT
TAG=round2 bash scripts/profile_r2.sh
cp gpurun_out/prof2/launches_round2.csv.gz $OUT/ 2>/dev/null
CMD="python scripts/bench_gemm.py am_lstm"
$CMD > $OUT/gemm_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 8 -c 1 \
    -o $OUT/full_gemm_am_lstm $CMD > $OUT/ncu_gemm.log 2>&1
echo "gemm full rc $?"
CMD="python bench.py --profile-only"
for spec in "lookahead_scores:100" "search_step:100" "att_context:100" "seg_scan:200" "pack_rows:1000" "copy_rows:200"; do
  k=${spec%%:*}; skip=${spec##*:}
  ncu --set full --clock-control none -k regex:$k --launch-skip $skip -c 1 \
      -o $OUT/full_$k $CMD > $OUT/ncu_$k.log 2>&1
  echo "full $k rc $?"
done
ls $OUT
