#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -s -x > gpurun_out/pytest_gpu.log 2>&1; grep -E "c2:|c5:|c4:|passed|failed|FAILED|rows vs|Error" gpurun_out/pytest_gpu.log | cut -c1-200 | head -8
for lib in libfusedbeam_b200_old.so libfusedbeam_b200.so; do
  FB_LIB_AB=$lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"row_norm|seg_sum" -s 50 -c 60 --csv python bench.py --profile-only 2>/dev/null | python -c "
import csv,sys
r=[x for x in csv.reader(sys.stdin) if len(x)>5]
h=r[0]; v=[float(x[h.index('Metric Value')].replace(',','')) for x in r[1:] if x[h.index('Metric Name')]=='gpu__time_duration.sum']
print('$lib row_norm', len(v), 'mean us', sum(v)/len(v)/1000 if v else None)"
done
for i in 1 2; do for lib in libfusedbeam_b200_old.so libfusedbeam_b200.so; do FB_LIB_AB=$lib timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b_ce.json 2>/dev/null; python -c "import json;j=json.load(open('gpurun_out/b_ce.json'));print('$lib', j['ms_per_step'], j['value'], 'e2e', j['e2e']['value'])"; done; done
