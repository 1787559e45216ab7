#!/bin/bash
FB_LIB_AB=libfusedbeam_b200_trace.so timeout 300 python scripts/rec_trace.py | grep -v "^ *[0-9]\{1,3\}  " | head -3
for lib in libfusedbeam_b200_d0.so libfusedbeam_b200.so; do echo "== $lib"; FB_LIB_AB=$lib timeout 300 python scripts/rec_trace.py; FB_LIB_AB=$lib FB_REC_KCB=5 timeout 300 python scripts/rec_trace.py; done
