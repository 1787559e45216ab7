#!/bin/bash
FB_LIB_AB=libfusedbeam_b200_trace.so timeout 300 python scripts/rec_trace.py | grep -v "^ *[0-9]\{1,3\}  " | head -7
for lib in libfusedbeam_b200_old.so libfusedbeam_b200.so; do echo "== $lib"; FB_LIB_AB=$lib timeout 300 python scripts/rec_trace.py; done
