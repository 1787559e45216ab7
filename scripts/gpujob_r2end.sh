#!/bin/bash
# round-end check as the driver runs it: smoke, the GPU suite, the default bench line
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_end.log 2>&1; tail -1 gpurun_out/pytest_gpu_end.log
timeout 1200 python bench.py > gpurun_out/end_bench.json 2> gpurun_out/end_bench.err; echo "bench rc $?"
python -c "import json;j=json.load(open('gpurun_out/end_bench.json'));print(j['value'], j['ms_per_step'], 'e2e', j['e2e']['value'], 'clocks', j['clocks'], 'cpu', j['cpu_baseline']['value'], j['cpu_baseline']['tokens_match_gpu'])"
