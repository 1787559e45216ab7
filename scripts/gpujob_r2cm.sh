#!/bin/bash
run() { env "$@" timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b_cm.json 2>/dev/null; python -c "import json;j=json.load(open('gpurun_out/b_cm.json'));print('$*', j['ms_per_step'], j['e2e']['tokens_equal_resident'])"; }
for i in 1 2; do
run FB_ATT_EW=8
run FB_ATT_EW=4
run FB_ATT_RE=6
done
