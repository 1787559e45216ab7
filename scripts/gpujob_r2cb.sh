#!/bin/bash
for k in 4 5 7 10; do echo "KCB=$k"; KCB=$k timeout 300 python scripts/bench_gemm.py lm_out_240 lm_out; done
