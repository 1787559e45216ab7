#!/bin/bash
# Full-size bench lines of the non-headline configurations (1 GPU):
#   c5: 4458 utterances (Switchboard-shaped, 30k-word look-ahead, beam 35)
#   c4: 2620 utterances (5k subword tokens, subword LM fusion, beam 60)
# each through the corpus path (length-sorted batches, fusion per batch).
mkdir -p gpurun_out
for spec in ${SPECS:-"c5:128" "c4:128"}; do
  cfg=${spec%%:*}; bs=${spec##*:}
  timeout ${TMO:-1500} python bench.py --config $cfg --batch $bs --steps ${STEPS:-2} \
      --warmup ${WARM:-3} --no-cpu-baseline ${EXTRA:-} > gpurun_out/bench_${cfg}_b${bs}.json \
      2> gpurun_out/bench_${cfg}_b${bs}.err
  echo "== $cfg batch $bs rc $?"
  tail -c 600 gpurun_out/bench_${cfg}_b${bs}.json; tail -2 gpurun_out/bench_${cfg}_b${bs}.err
done
