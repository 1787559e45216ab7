#!/bin/bash
FB_LIB_AB=libfusedbeam_b200_traces.so KCB=1 SLOT=1 timeout 300 python scripts/gemm_trace.py | tail -5
for lib in libfusedbeam_b200.so libfusedbeam_b200_spin.so; do echo "== $lib"; FB_LIB_AB=$lib KCB=1 timeout 300 python scripts/bench_gemm.py am_lstm am_lstm_2k lm_lstm; done
