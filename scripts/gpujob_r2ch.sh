#!/bin/bash
SPECS="c5:256 c4:256" timeout 1500 bash scripts/bench_configs.sh > gpurun_out/configs.log 2>&1
for c in c5 c4; do python -c "import json;j=json.load(open('gpurun_out/bench_${c}_b256.json'));print('$c', j['value'], 'e2e', j['e2e']['value'], j['ms_per_step'])"; done
