#!/bin/bash
for lib in trace trace1 trace2; do echo "== $lib"; FB_LIB_AB=libfusedbeam_b200_$lib.so timeout 300 python scripts/rec_trace.py | grep -v "^ *[0-9]"; done
for lib in libfusedbeam_b200.so libfusedbeam_b200_p1.so libfusedbeam_b200_p2.so; do echo "== $lib"; FB_LIB_AB=$lib timeout 300 python scripts/rec_trace.py; done
