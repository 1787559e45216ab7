#!/bin/bash
# Round-2 launch list of one c2 decode with per-launch DRAM bytes and tensor
# pipe activity (run under gpurun; the plain run must exit 0 first).
set -u
OUT=gpurun_out/prof2
mkdir -p $OUT
CMD="python bench.py --profile-only ${PROF_ARGS:-}"
$CMD > $OUT/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
    --clock-control none --csv --log-file $OUT/launches_${TAG:-c2}.csv $CMD > $OUT/ncu.log 2>&1
echo "launch list rc $?"
gzip -f $OUT/launches_${TAG:-c2}.csv
