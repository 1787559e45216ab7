#!/bin/bash
for lib in libfusedbeam_b200_g1.so libfusedbeam_b200.so libfusedbeam_b200_g4.so; do echo "== $lib"; for k in 1 4; do FB_LIB_AB=$lib KCB=$k timeout 300 python scripts/bench_gemm.py am_lstm am_lstm_2k lm_lstm lm_out_240; done; done
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x 2>&1 | tail -2
FB_LIB_AB=libfusedbeam_b200_g4.so timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x 2>&1 | tail -2
