#!/bin/bash
# 128- vs 64-wide GEMM tiles after the TMA-store epilogue: graph-timed
# per-shape GEMMs, then the c2 decode under each setting.
S="lm_lstm_64 lm_lstm_160 lm_lstm lm_lstm_300 lm_lstm_600 am_lstm_2k am_lstm am_q enc_rec"
for bn in "" 64; do
  echo "== FB_GEMM_BN=$bn"
  FB_GEMM_BN=$bn timeout 300 python scripts/bench_gemm.py $S 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.rstrip()); continue
    print(d.get('name', d.get('shape')), {k: v for k, v in d.items() if 'us' in k or k in ('tflops',)})"
done
bash scripts/sweep_env.sh "" "FB_GEMM_BN=64" "" "FB_GEMM_BN=64"
