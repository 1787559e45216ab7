#!/bin/bash
# tail regime: a 16-utterance c2 batch (every step has few live rows)
timeout 600 python bench.py --utts 16 --no-cpu-baseline --steps 5 --warmup 3 --stats > gpurun_out/b_tail.json 2> gpurun_out/b_tail.err
python -c "import json;j=json.load(open('gpurun_out/b_tail.json'));print('16 utts', j['ms_per_step'], 'steps', j.get('decode_steps_mean'))"
grep -i "steps\|step" gpurun_out/b_tail.err | tail -3
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_tail.csv python bench.py --profile-only --utts 16 > /dev/null 2>&1; echo "ncu rc $?"
gzip -f gpurun_out/launches_tail.csv
