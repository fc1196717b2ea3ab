# A/B of the (leaf half, vector chunk) split of k_leaf_dense_split: parity (on), cfg3s and cfg2 both ways
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_leaf.log 2>&1; echo pytest=$? >> gpurun_out/pytest_leaf.log
for cfg in cfg3s cfg2; do
  for sp in 1 0; do
    H2_LEAF_VSPLIT=$sp timeout 300 python bench.py --config $cfg --steps 20 --no-cpu-baseline --no-e2e > gpurun_out/ab_${cfg}_$sp.json 2>gpurun_out/ab_${cfg}_$sp.err
    python -c "
import json; d=json.load(open('gpurun_out/ab_${cfg}_$sp.json'))
print('$cfg split=$sp', round(d['value']), [round(v['ms_per_matvec'],4) for v in d['per_nv'].values()])
for k,v in d['per_nv'].items(): print(k, {a: round(x*1000,1) for a,x in v['phases_ms'].items()})
" >> gpurun_out/ab_leaf.txt
  done
done
