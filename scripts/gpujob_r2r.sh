#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/rec_trace.py
FB_REC_KCB=5 timeout 300 python scripts/rec_trace.py
B=256 timeout 300 python scripts/rec_trace.py
FB_LIB_AB=libfusedbeam_b200_trace.so timeout 300 python scripts/rec_trace.py
