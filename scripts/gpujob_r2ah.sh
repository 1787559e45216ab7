#!/bin/bash
mkdir -p gpurun_out
PROF_ARGS="" TAG=c2 bash scripts/profile_r2.sh
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lstm_rec -c 1 \
  -o gpurun_out/round2_full_lstm_rec python bench.py --profile-only > gpurun_out/ncu_rec.log 2>&1
echo "rec capture rc $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:att_energy -s 40 -c 1 \
  -o gpurun_out/round2_full_att_energy python bench.py --profile-only > gpurun_out/ncu_en.log 2>&1
echo "energy capture rc $?"
