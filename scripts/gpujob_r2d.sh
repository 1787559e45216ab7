#!/bin/bash
# round-2 GPU job d: precision sources of the long-decode score drift (c5/c4):
# default vs precise LSTM activations vs bf16x3 operands, against the fp64 oracle
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py -m gpu -q -x > gpurun_out/pytest_gemm.log 2>&1; tail -2 gpurun_out/pytest_gemm.log
for c in c5 c4; do
  timeout 300 python scripts/parity_dump.py $c d > /dev/null 2>&1
  FB_LIB_AB=libfusedbeam_b200_precise.so timeout 300 python scripts/parity_dump.py $c precise > /dev/null 2>&1
done
t() { python -c "import json;j=json.load(open('gpurun_out/$1.json'));print('$1', j['ms_per_step'], 'e2e', j['e2e']['value'], 'frac', j['roofline']['frac'], 'gemm ms', j['roofline']['gemm_ms_per_decode'])"; }
timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/b_d.json 2> gpurun_out/b_d.err; t b_d
FB_LIB_AB=libfusedbeam_b200_precise.so timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/b_precise.json 2> gpurun_out/b_precise.err; t b_precise
ls gpurun_out | head -50
