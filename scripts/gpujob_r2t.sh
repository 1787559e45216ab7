#!/bin/bash
FB_LIB_AB=libfusedbeam_b200_trace.so timeout 300 python scripts/rec_trace.py
timeout 900 python -m pytest tests/test_gpu_parity_full.py -q -s -x 2>&1 | grep -E "utterances|passed|failed"
