#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -s -x > gpurun_out/pytest_gpu.log 2>&1; grep -E "utterances|passed|failed|FAILED|rows vs|Error|assert" gpurun_out/pytest_gpu.log | head -14
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b_bg$i.json 2>/dev/null; python -c "import json;j=json.load(open('gpurun_out/b_bg$i.json'));print('bg$i', j['ms_per_step'], j['value'], 'e2e', j['e2e']['value'])"; done
