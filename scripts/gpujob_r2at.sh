#!/bin/bash
for lib in libfusedbeam_b200.so libfusedbeam_b200_nod.so; do echo "== $lib"; FB_LIB_AB=$lib KCB=1 timeout 300 python scripts/bench_gemm.py am_lstm lm_out_240; done
