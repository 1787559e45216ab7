#!/bin/bash
# round-2 GPU job j: register caps (no spills), tail stream-K A/B, per-step times
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_models.py tests/test_gpu_search.py -m gpu -q > gpurun_out/pytest_j.log 2>&1; tail -1 gpurun_out/pytest_j.log
timeout 600 python -m pytest tests/test_gpu_parity_full.py -m gpu -q -s -k "c2 or c5" > gpurun_out/parity_j.log 2>&1; grep -E "utterances|passed|failed" gpurun_out/parity_j.log
t() { python -c "import json;j=json.load(open('gpurun_out/$1.json'));print('$1', j['ms_per_step'], 'e2e', j['e2e']['value'], 'frac', j['roofline']['frac'])"; }
for v in "base:" "tsk:FB_TAIL_SPLITK=1" "lsk:FB_LM_SPLITK=1" "base2:"; do
  tag=${v%%:*}; envs=${v#*:}
  env $envs timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b_$tag.json 2>/dev/null; t b_$tag
done
timeout 300 python scripts/step_times.py > gpurun_out/step_times.log 2>&1; tail -12 gpurun_out/step_times.log
