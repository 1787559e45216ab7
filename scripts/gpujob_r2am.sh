#!/bin/bash
for k in 1 2 4 16; do echo "KCB=$k"; KCB=$k timeout 300 python scripts/bench_gemm.py am_lstm am_lstm_2k lm_lstm; done
