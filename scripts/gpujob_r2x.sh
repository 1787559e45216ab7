#!/bin/bash
FB_LIB_AB=libfusedbeam_b200_tracex.so timeout 300 python scripts/rec_trace.py | grep -v "^ *[0-9]\{1,3\}  " | head -9
