#!/bin/bash
# round-2 GPU job f: fp64 normalisers + decoder-LSTM TMEM chunks: tests, parity, drift, timing
mkdir -p gpurun_out
timeout 300 python scripts/stats_debug.py > gpurun_out/stats_debug.log 2>&1; cat gpurun_out/stats_debug.log | tail -5
timeout 900 python -m pytest tests -m gpu -q --deselect tests/test_gpu_parity_full.py > gpurun_out/pytest_gpu.log 2>&1; grep -E "passed|failed|FAILED" gpurun_out/pytest_gpu.log | head -8
timeout 600 python -m pytest tests/test_gpu_parity_full.py -m gpu -q -s > gpurun_out/parity_all.log 2>&1; grep -E "utterances|passed|failed" gpurun_out/parity_all.log
for c in c2 c4 c5; do timeout 300 python scripts/parity_dump.py $c f > /dev/null 2>&1; done
timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/b_f.json 2> gpurun_out/b_f.err; python -c "import json;j=json.load(open('gpurun_out/b_f.json'));print('f', j['ms_per_step'], j['e2e']['value'], j['roofline']['frac'])"
