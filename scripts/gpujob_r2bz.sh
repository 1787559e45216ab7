#!/bin/bash
run() { env "$@" timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b_bz.json 2>/dev/null; python -c "import json;j=json.load(open('gpurun_out/b_bz.json'));print('$*', j['ms_per_step'])"; }
for i in 1 2; do
run FB_TAIL_TILING=4,4,160
run FB_TAIL_TILING=4,4,32
run FB_TAIL_TILING=4,4,16
run FB_TAIL_TILING=2,4,32
run FB_TAIL_TILING=2,4,16
done
