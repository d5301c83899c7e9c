# quick decode measurement: bench.py default without the CPU leg, one line per mode
python bench.py --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))
for k,v in d['per_mode'].items(): print(k, round(v['decode_tok_s'],1), 'tok/s', round(v['hbm_frac_of_measured'],4), 'prefill_ms', round(v['prefill_ms'],2))
"
