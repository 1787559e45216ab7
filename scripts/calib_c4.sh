# c4 calibration sweep (random-init model): decode length / finishing vs output scales
for a in ${A:-1.0 1.5}; do for e in ${E:-0.5 1.0 1.5}; do for l in ${L:-0.25 0.5}; do
echo "== asr.out_scale=$a asr.eos_bias=$e sublm.out_scale=$l"
timeout 300 python bench.py --config c4 --utts ${UTTS:-8} --steps 1 --warmup 1 --no-cpu-baseline --stats --set asr.out_scale=$a --set asr.eos_bias=$e --set sublm.out_scale=$l 2>&1 | python -c "
import sys,json
for line in sys.stdin:
    if line.startswith('{'):
        j=json.loads(line); print('  ms', j['ms_per_step'], 'steps', j['decode_steps_mean'], 'fin', j['finished_frac'])
    elif 'distinct' in line or line.startswith('utt'): print('  ', line.rstrip()[:100])
"
done; done; done
