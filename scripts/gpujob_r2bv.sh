#!/bin/bash
for lib in libfusedbeam_b200_old.so libfusedbeam_b200.so; do
  FB_LIB_AB=$lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:boundary_plan -s 50 -c 40 --csv python bench.py --profile-only 2>/dev/null | python -c "
import csv,sys
r=[x for x in csv.reader(sys.stdin) if len(x)>5]
h=r[0]; v=[float(x[h.index('Metric Value')].replace(',','')) for x in r[1:] if x[h.index('Metric Name')]=='gpu__time_duration.sum']
print('$lib', len(v), 'mean us', sum(v)/len(v)/1000 if v else None)"
done
