#!/bin/bash
FB_LIB_AB=libfusedbeam_b200_trace.so timeout 300 python scripts/rec_trace.py | grep -v "^ *[0-9]\{1,3\}  " | head -3
for lib in libfusedbeam_b200_old.so libfusedbeam_b200.so; do echo "== $lib"; FB_LIB_AB=$lib KCB=1 timeout 300 python scripts/bench_gemm.py am_lstm lm_lstm am_lstm_2k; FB_LIB_AB=$lib timeout 300 python scripts/rec_trace.py; done
timeout 900 python -m pytest tests -m gpu -q -s -x > gpurun_out/pytest_gpu.log 2>&1; grep -E "utterances|passed|failed|FAILED|rows vs" gpurun_out/pytest_gpu.log | head -12
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b_ae$i.json 2>/dev/null; python -c "import json;j=json.load(open('gpurun_out/b_ae$i.json'));print('ae$i', j['ms_per_step'], j['value'], 'e2e', j['e2e']['value'])"; done
FB_LIB_AB=libfusedbeam_b200_old.so timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b_ae0.json 2>/dev/null; python -c "import json;j=json.load(open('gpurun_out/b_ae0.json'));print('old', j['ms_per_step'], j['value'], 'e2e', j['e2e']['value'])"
