#!/bin/bash
# Round profiling + summaries on the GPU box, keeping gpurun_out/ under the
# 64 MiB merge limit: bench line, launch list (gzip), ncu summaries; only the
# GEMM and energy-kernel reports are kept.
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
bash scripts/profile_round.sh > gpurun_out/prof.log 2>&1
python scripts/launch_summary.py gpurun_out/prof/launches_c2.csv > gpurun_out/prof/launches_summary.txt 2>&1
python scripts/ncu_summary.py gpurun_out/prof/full_gemm_tc_kernel.ncu-rep gpurun_out/prof/full_att_energy.ncu-rep \
  gpurun_out/prof/full_att_context.ncu-rep gpurun_out/prof/full_pack_rows.ncu-rep \
  gpurun_out/prof/full_search_step.ncu-rep gpurun_out/prof/full_spec_select.ncu-rep \
  gpurun_out/prof/full_seg_scan.ncu-rep gpurun_out/prof/full_seg_sum.ncu-rep > gpurun_out/prof/full_summary.csv 2>&1
gzip -f gpurun_out/prof/launches_c2.csv
for f in gpurun_out/prof/full_*.ncu-rep; do
  case $f in *gemm_tc_kernel*|*att_energy*) ;; *) rm -f $f ;; esac
done
du -sh gpurun_out
