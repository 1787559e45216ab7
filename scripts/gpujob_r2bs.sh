#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -s -x > gpurun_out/pytest_gpu.log 2>&1; grep -E "c2:|c5:|c4:|passed|failed|FAILED|rows vs" gpurun_out/pytest_gpu.log | cut -c1-200 | head -8
for lib in libfusedbeam_b200_q0.so libfusedbeam_b200.so; do echo "== $lib"; FB_LIB_AB=$lib timeout 300 python scripts/bench_attention.py; done
for i in 1 2; do for lib in libfusedbeam_b200_q0.so libfusedbeam_b200.so; do FB_LIB_AB=$lib timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b_bs.json 2>/dev/null; python -c "import json;j=json.load(open('gpurun_out/b_bs.json'));print('$lib', j['ms_per_step'], j['value'], 'e2e', j['e2e']['value'])"; done; done
