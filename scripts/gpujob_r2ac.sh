#!/bin/bash
FB_LIB_AB=libfusedbeam_b200_trace.so timeout 300 python scripts/rec_trace.py | grep -v "^ *[0-9]\{1,3\}  " | head -3
for w in 1 3 7; do echo "== wide $w"; FB_REC_WIDE=$w timeout 300 python scripts/rec_trace.py; done
timeout 900 python -m pytest tests -m gpu -q -s -x > gpurun_out/pytest_gpu.log 2>&1; grep -E "utterances|passed|failed|FAILED|rows vs" gpurun_out/pytest_gpu.log | head -12
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b_ac$i.json 2>/dev/null; python -c "import json;j=json.load(open('gpurun_out/b_ac$i.json'));print('ac$i', j['ms_per_step'], j['value'], 'e2e', j['e2e']['value'])"; done
