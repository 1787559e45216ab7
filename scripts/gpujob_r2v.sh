#!/bin/bash
FB_LIB_AB=libfusedbeam_b200_trace.so timeout 300 python scripts/rec_trace.py | grep -v "^ *[0-9]\{1,3\}  "
