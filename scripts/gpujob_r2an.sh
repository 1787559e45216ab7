#!/bin/bash
for k in 1 16; do echo "== KCB=$k"; FB_LIB_AB=libfusedbeam_b200_trace.so KCB=$k timeout 300 python scripts/gemm_trace.py; done
