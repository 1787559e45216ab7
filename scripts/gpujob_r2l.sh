#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_models.py -m gpu -q -x 2>&1 | tail -2
echo "== default"; python scripts/bench_gemm.py lm_out_240 lm_out am_lstm am_lstm_2k lm_lstm_160
echo "== KCB=1"; KCB=1 python scripts/bench_gemm.py lm_out_240 am_lstm am_lstm_2k
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b_l$i.json 2>/dev/null; python -c "import json;j=json.load(open('gpurun_out/b_l$i.json'));print('l$i', j['ms_per_step'], 'e2e', j['e2e']['value'])"; done
