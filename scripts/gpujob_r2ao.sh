#!/bin/bash
FB_LIB_AB=libfusedbeam_b200_traces.so KCB=1 SLOT=1 timeout 300 python scripts/gemm_trace.py
