#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x 2>&1 | tail -1
bash scripts/gpujob_r2bf.sh
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b_bi$i.json 2>/dev/null; python -c "import json;j=json.load(open('gpurun_out/b_bi$i.json'));print('bi$i', j['ms_per_step'], j['value'], 'e2e', j['e2e']['value'])"; done
