#!/bin/bash
# round-2 GPU job h: recurrence TMEM chunks (drift + timing)
mkdir -p gpurun_out
for c in c4 c5; do timeout 300 python scripts/parity_dump.py $c h > /dev/null 2>&1; done
FB_REC_KCB=2 timeout 300 python scripts/parity_dump.py c4 h2 > /dev/null 2>&1
timeout 600 python scripts/step_error.py c4 1822 > gpurun_out/step_error_c4h.log 2>&1; tail -9 gpurun_out/step_error_c4h.log | head -3
for v in "r1:FB_REC_KCB=1" "r2:FB_REC_KCB=2" "rall:FB_REC_KCB=64"; do
  tag=${v%%:*}; envs=${v#*:}
  env $envs timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/b_$tag.json 2>/dev/null
  python -c "import json;j=json.load(open('gpurun_out/b_$tag.json'));print('$tag', j['ms_per_step'])"
done
timeout 300 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_models.py -m gpu -q > gpurun_out/pytest_gm.log 2>&1; tail -1 gpurun_out/pytest_gm.log
