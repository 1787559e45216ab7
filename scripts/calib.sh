# calibration sweep of a random-init workload: decode length / finishing vs scales
#   CFG=c5 UTTS=128 SETS="asr.out_scale=1.5,asr.eos_bias=-2 asr.out_scale=2,asr.eos_bias=-3" bash scripts/calib.sh
for s in $SETS; do
echo "== $CFG $s"
args=""; for kv in $(echo $s | tr ',' ' '); do args="$args --set $kv"; done
timeout 300 python bench.py --config $CFG --utts ${UTTS:-128} --steps 1 --warmup 1 --no-cpu-baseline --stats $args $EXTRA 2>&1 | python -c "
import sys,json
for line in sys.stdin:
    if line.startswith('{'):
        j=json.loads(line); print('  ms', j['ms_per_step'], 'steps', j['decode_steps_mean'], 'fin', j['finished_frac'])
    elif 'distinct' in line or line.startswith('utt'): print('  ', line.rstrip()[:100])
    elif 'Error' in line or 'error' in line: print('  ', line.rstrip()[:200])
"
done
