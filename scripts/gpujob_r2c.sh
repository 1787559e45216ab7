#!/bin/bash
# round-2 GPU job c: 256-wide tiles + GEMM bias diagnostics + A/B timing
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py -m gpu -q -x > gpurun_out/pytest_gemm.log 2>&1; tail -3 gpurun_out/pytest_gemm.log
timeout 300 python scripts/gemm_bias.py > gpurun_out/gemm_bias.log 2>&1; cat gpurun_out/gemm_bias.log | tail -5
t() { python -c "import json;j=json.load(open('gpurun_out/$1.json'));print('$1', j['ms_per_step'], 'e2e', j['e2e']['value'], 'frac', j['roofline']['frac'], 'gemm ms', j['roofline']['gemm_ms_per_decode'])"; }
for v in "default:" "n256:FB_GEMM_256=0" "noseg:FB_SEG_FUSED=0" "default2:"; do
  tag=${v%%:*}; env=${v#*:}
  env $env timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/b_$tag.json 2> gpurun_out/b_$tag.err; t b_$tag
done
timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_parity_full.py > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python -m pytest tests/test_gpu_parity_full.py -m gpu -q -s > gpurun_out/parity_all.log 2>&1; grep -E "utterances|passed|failed" gpurun_out/parity_all.log; for c in c2 c4 c5; do timeout 300 python scripts/parity_dump.py $c f64out > /dev/null 2>&1; done
