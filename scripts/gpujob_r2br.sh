#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_models.py -q -x 2>&1 | tail -1
for lib in libfusedbeam_b200_old.so libfusedbeam_b200.so; do echo "== $lib"; FB_LIB_AB=$lib timeout 300 python scripts/bench_gemm.py lm_out_240 lm_lstm am_lstm enc_proj; done
for i in 1 2; do for lib in libfusedbeam_b200_old.so libfusedbeam_b200.so; do FB_LIB_AB=$lib timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b_br.json 2>/dev/null; python -c "import json;j=json.load(open('gpurun_out/b_br.json'));print('$lib', j['ms_per_step'], j['value'], 'e2e', j['e2e']['value'])"; done; done
