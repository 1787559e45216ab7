#!/bin/bash
timeout 300 python scripts/bench_gemm.py lm_out lm_out_240
FB_GEMM_TMA_STORE=0 timeout 300 python scripts/bench_gemm.py lm_out lm_out_240
FB_LIB_AB=libfusedbeam_b200_trace.so SHAPE=240,65003,1216 MODE=0 KCB=0 SEGS=4 timeout 300 python scripts/gemm_trace.py | tail -5
