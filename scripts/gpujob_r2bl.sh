#!/bin/bash
FB_LIB_AB=libfusedbeam_b200_trace.so SHAPE=240,65003,1216 MODE=2 KCB=0 SEGS=8 timeout 300 python scripts/gemm_trace.py | tail -30
