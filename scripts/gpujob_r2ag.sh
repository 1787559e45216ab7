#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -s -x > gpurun_out/pytest_gpu.log 2>&1; grep -E "utterances|passed|failed|FAILED|rows vs" gpurun_out/pytest_gpu.log | head -12
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b_ag$i.json 2>/dev/null; python -c "import json;j=json.load(open('gpurun_out/b_ag$i.json'));print('ag$i', j['ms_per_step'], j['value'], 'e2e', j['e2e']['value'])"; done
SPECS="c5:256 c4:256" timeout 1200 bash scripts/bench_configs.sh > gpurun_out/configs.log 2>&1; for c in c5 c4; do python -c "import json;j=json.load(open('gpurun_out/bench_${c}_b256.json'));print('$c', j['value'], 'e2e', j['e2e']['value'])"; done
