# A/B of library variants built by tools/build_variants.sh on whole cycles (the copy on the GPU box is scratch)
cp paper_2509_06744_b200/libbmgcuda.so /tmp/libbmgcuda_keep.so
for spec in "$@"; do   # variant or variant:BMG_SYM_COLMAP value
  v=${spec%%:*}; cm=0; [ "$spec" != "$v" ] && cm=${spec#*:}
  echo "== variant $v colmap $cm"
  cp paper_2509_06744_b200/variants/libbmgcuda_$v.so paper_2509_06744_b200/libbmgcuda.so
  BMG_SYM_COLMAP=$cm python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-parity --no-batch 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('C4', round(d['value'],3), 'V/s', round(d['ms_per_step'],3), 'ms', d['clocks']['sm_mhz'], 'MHz', 'roofline pass', round(d['roofline']['half_storage_pass_ms'],4))
for k,e in d['extra_configs'].items():
    if 'value' in e: print(k, round(e['value'],3), e.get('unit'), e.get('ms_per_step', e.get('ms')), e.get('clocks',{}).get('sm_mhz'))
    else: print(k, e)
"
done
cp /tmp/libbmgcuda_keep.so paper_2509_06744_b200/libbmgcuda.so
