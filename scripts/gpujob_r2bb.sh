#!/bin/bash
for i in 1 2; do for v in late0 late1 main0; do
  case $v in late0) lib=libfusedbeam_b200_late.so; p=1;; late1) lib=libfusedbeam_b200_late.so; p=1;; main0) lib=libfusedbeam_b200.so; p=0;; esac
  FB_LIB_AB=$lib FB_PDL=$p timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b_bb.json 2>/dev/null; python -c "import json;j=json.load(open('gpurun_out/b_bb.json'));print('$v', j['ms_per_step'], j['value'], 'e2e', j['e2e']['value'])"; done; done
