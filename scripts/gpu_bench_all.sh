#!/bin/bash
# Round-end bench lines: c2 (headline, default) and c4 (subword, 32 utterances)
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo c2=$?
timeout 900 python bench.py --config c4 --utts 32 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4=$?
head -c 400 gpurun_out/bench_c2.json; echo; head -c 400 gpurun_out/bench_c4.json
