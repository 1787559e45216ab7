#!/bin/bash
# round-2 GPU job: build check, tests, full-set parity, dumps, A/B timing of the
# operand formats, per-step error trace, c4/c5 full-size bench lines
mkdir -p gpurun_out
python -c "import paper_1909_08723_b200.kernels as K; print('operand format', K.operand_format())"
timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_parity_full.py > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python -m pytest tests/test_gpu_parity_full.py -m gpu -q -s > gpurun_out/parity_fp16.log 2>&1; grep -E "utterances|passed|failed|assert " gpurun_out/parity_fp16.log | head -12
for c in c2 c4 c5; do timeout 300 python scripts/parity_dump.py $c fp16 > /dev/null 2>&1; FB_LIB_AB=libfusedbeam_b200_bf16x3.so timeout 300 python scripts/parity_dump.py $c bf16 > /dev/null 2>&1; done
timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench_fp16.json 2> gpurun_out/bench_fp16.err; python -c "import json;j=json.load(open('gpurun_out/bench_fp16.json'));print('fp16', j['ms_per_step'], j['e2e']['value'], j['roofline']['frac'], j['roofline']['gemm_ms_per_decode'])"
FB_LIB_AB=libfusedbeam_b200_bf16x3.so timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench_bf16.json 2> gpurun_out/bench_bf16.err; python -c "import json;j=json.load(open('gpurun_out/bench_bf16.json'));print('bf16', j['ms_per_step'], j['e2e']['value'], j['roofline']['frac'], j['roofline']['gemm_ms_per_decode'])"
timeout 300 python scripts/step_error.py c4 1822 > gpurun_out/step_error_c4.log 2>&1; tail -8 gpurun_out/step_error_c4.log
SPECS="c5:128 c4:32 c4:128" STEPS=2 WARM=3 bash scripts/bench_configs.sh
ls gpurun_out
