#!/bin/bash
# round-2 GPU job i: full validation, bench lines (c2 + reference arm, c5, c4), launch list
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu.log 2>&1; grep -E "utterances|passed|failed|FAILED" gpurun_out/pytest_gpu.log | head -12
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -c 400 gpurun_out/bench_c2.json; echo
timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref_c2.json 2> gpurun_out/ref_c2.err; tail -c 300 gpurun_out/ref_c2.json; echo
SPECS="c5:128 c5:256 c4:128 c4:256" STEPS=2 WARM=3 bash scripts/bench_configs.sh > gpurun_out/bench_configs.log 2>&1; grep "==" gpurun_out/bench_configs.log
TAG=round2 bash scripts/profile_r2.sh
ls gpurun_out/prof2
