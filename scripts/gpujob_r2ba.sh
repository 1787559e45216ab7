#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -s -x > gpurun_out/pytest_gpu.log 2>&1; grep -E "utterances|passed|failed|FAILED|rows vs|Error" gpurun_out/pytest_gpu.log | head -12
for i in 1 2; do for v in 1 0; do FB_PDL=$v timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b_ba.json 2>gpurun_out/b_ba.err; python -c "import json;j=json.load(open('gpurun_out/b_ba.json'));print('pdl $v', j['ms_per_step'], j['value'], 'e2e', j['e2e']['value'])" || tail -3 gpurun_out/b_ba.err; done; done
