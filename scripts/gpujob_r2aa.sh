#!/bin/bash
for lib in trace; do echo "== $lib"; FB_LIB_AB=libfusedbeam_b200_$lib.so timeout 300 python scripts/rec_trace.py | grep -v "^ *[0-9]\{1,3\}  " | head -9; done
for lib in libfusedbeam_b200_p0.so libfusedbeam_b200_l0.so libfusedbeam_b200.so; do echo "== $lib"; FB_LIB_AB=$lib timeout 300 python scripts/rec_trace.py; done
