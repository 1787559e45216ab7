#!/bin/bash
mkdir -p gpurun_out
S="lm_out_240 lm_out lm_lstm_160 lm_lstm_64 am_lstm am_lstm_2k am_q enc_proj"
echo "== default"; python scripts/bench_gemm.py $S
echo "== KCB=1"; KCB=1 python scripts/bench_gemm.py lm_out_240 am_lstm am_lstm_2k
echo "== bf16x3"; FB_LIB_AB=libfusedbeam_b200_bf16x3.so python scripts/bench_gemm.py $S
