#!/bin/bash
# critical-path probe: duplicate one idempotent kernel per step (dev builds)
for i in 1 2; do for lib in libfusedbeam_b200.so libfusedbeam_b200_dctx.so libfusedbeam_b200_dscan.so; do FB_LIB_AB=$lib timeout 600 python bench.py --no-cpu-baseline --steps 6 --warmup 3 > gpurun_out/b_aj.json 2>/dev/null; python -c "import json;j=json.load(open('gpurun_out/b_aj.json'));print('$lib', j['ms_per_step'])"; done; done
