# A/B of an environment switch on whole cycles: bash tools/ab_env.sh VAR v1 v2 ... -> C4, C2, C3@512, C5@1024 V-cycles/s per value
var=$1; shift
for v in "$@"; do
  echo "== $var=$v"
  env $var=$v python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-parity --no-batch 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('C4', round(d['value'],3), 'V/s', round(d['ms_per_step'],3), 'ms', d['clocks']['sm_mhz'], 'MHz', 'roofline pass', round(d['roofline']['half_storage_pass_ms'],4))
for k,e in d['extra_configs'].items():
    if 'value' in e: print(k, round(e['value'],3), e.get('unit'), e.get('ms_per_step', e.get('ms')), e.get('clocks',{}).get('sm_mhz'))
    else: print(k, e)
"
done
