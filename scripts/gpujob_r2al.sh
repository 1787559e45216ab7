#!/bin/bash
for i in 1 2; do for sp in 2 4; do FB_ATT_SPLIT=$sp timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b_al.json 2>/dev/null; python -c "import json;j=json.load(open('gpurun_out/b_al.json'));print('split $sp', j['ms_per_step'], j['value'], 'e2e', j['e2e']['value'])"; done; done
