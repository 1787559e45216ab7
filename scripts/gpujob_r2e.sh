#!/bin/bash
# round-2 GPU job e: which GEMM family's TMEM accumulation chunk carries the drift
mkdir -p gpurun_out
for v in "am:FB_KCB_AM=1" "enc:FB_KCB_ENC=1" "lm:FB_KCB_LM=1" "amenc:FB_KCB_AM=1 FB_KCB_ENC=1"; do
  tag=${v%%:*}; envs=${v#*:}
  env $envs timeout 300 python scripts/parity_dump.py c5 k$tag > /dev/null 2>&1
  env $envs timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/b_k$tag.json 2>/dev/null
  python -c "import json;j=json.load(open('gpurun_out/b_k$tag.json'));print('$tag', j['ms_per_step'])"
done
env FB_KCB_AM=1 FB_KCB_ENC=1 timeout 300 python scripts/parity_dump.py c4 kamenc > /dev/null 2>&1
env FB_KCB_AM=1 FB_KCB_ENC=1 timeout 300 python scripts/parity_dump.py c2 kamenc > /dev/null 2>&1
