#!/bin/bash
mkdir -p gpurun_out
for k in 2; do
  FB_KCB_AM=$k timeout 300 python scripts/parity_dump.py c5 kam$k > /dev/null 2>&1
  FB_KCB_AM=$k timeout 300 python scripts/parity_dump.py c2 kam$k > /dev/null 2>&1
  FB_KCB_AM=$k timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b_kam$k.json 2>/dev/null; python -c "import json;j=json.load(open('gpurun_out/b_kam$k.json'));print('kam$k', j['ms_per_step'], 'e2e', j['e2e']['value'])"
done
timeout 300 python scripts/parity_dump.py c5 m1 > /dev/null 2>&1
KCB=2 python scripts/bench_gemm.py am_lstm am_lstm_2k
