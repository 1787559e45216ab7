#!/bin/bash
for i in 1 2; do for cq in 160 80 54; do FB_ATT_CQ=$cq timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b_ax.json 2>/dev/null; python -c "import json;j=json.load(open('gpurun_out/b_ax.json'));print('cq $cq', j['ms_per_step'], j['value'], 'e2e', j['e2e']['value'])"; done; done
