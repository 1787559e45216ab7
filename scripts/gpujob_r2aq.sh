#!/bin/bash
FB_LIB_AB=libfusedbeam_b200_tracec.so KCB=1 COMMIT=1 timeout 300 python scripts/gemm_trace.py | sed -n '1,12p;42,70p'
