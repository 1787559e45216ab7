#!/bin/bash
FB_GEMM_TMA_STORE=0 FB_LIB_AB=libfusedbeam_b200_nost.so SHAPE=240,65003,1216 MODE=0 KCB=0 SEGS=2 timeout 300 python scripts/gemm_trace.py | tail -4
FB_GEMM_TMA_STORE=0 FB_LIB_AB=libfusedbeam_b200_nost.so timeout 300 python scripts/bench_gemm.py lm_out
FB_GEMM_TMA_STORE=0 timeout 300 python scripts/bench_gemm.py lm_out
