#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_launch_modes.py -q -x 2>&1 | tail -3
