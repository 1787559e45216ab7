# c5 calibration sweep (random-init model): decode length / finishing vs output scales
# (the LM scales follow c2's: emb 0.2, </s> bias 5, LSTM range x2)
for a in ${A:-0.7}; do for e in ${E:--1.5 -0.75 0}; do
echo "== asr.out_scale=$a asr.eos_bias=$e"
timeout 300 python bench.py --config c5 --utts ${UTTS:-128} --steps 1 --warmup 1 --no-cpu-baseline --stats --set asr.out_scale=$a --set asr.eos_bias=$e --set lm.emb_scale=0.2 --set lm.eos_bias=5 --set lm.w_scale=2 2>&1 | python -c "
import sys,json
for line in sys.stdin:
    if line.startswith('{'):
        j=json.loads(line); print('  ms', j['ms_per_step'], 'steps', j['decode_steps_mean'], 'fin', j['finished_frac'])
    elif 'distinct' in line or line.startswith('utt'): print('  ', line.rstrip()[:100])
    elif 'Error' in line or 'error' in line: print('  ', line.rstrip()[:200])
"
done; done
