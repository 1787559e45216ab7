#!/bin/bash
mkdir -p gpurun_out
for v in "f1:" "f0:FB_SEG_FOLD=0" "f1b:" "f0b:FB_SEG_FOLD=0"; do
  tag=${v%%:*}; envs=${v#*:}
  env $envs timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b_$tag.json 2>/dev/null
  python -c "import json;j=json.load(open('gpurun_out/b_$tag.json'));print('$tag', j['ms_per_step'], 'e2e', j['e2e']['value'])"
done
