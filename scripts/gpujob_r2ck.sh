#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -s -x > gpurun_out/pytest_gpu.log 2>&1; grep -E "c2:|c5:|c4:|passed|failed|FAILED|rows vs|Error|assert" gpurun_out/pytest_gpu.log | cut -c1-200 | head -8
for i in 1 2 3; do timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b_ck.json 2>/dev/null; python -c "import json;j=json.load(open('gpurun_out/b_ck.json'));print('ck', j['ms_per_step'], j['value'], 'e2e', j['e2e']['value'], j['e2e']['tokens_equal_resident'])"; done
