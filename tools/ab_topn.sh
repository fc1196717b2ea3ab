# A/B of the fused single-CTA top sweep levels (H2_TOPN=8 default vs 0 = one launch per level)
for cfg in cfg3s cfg2; do
  for tn in 8 0 2; do
    H2_TOPN=$tn timeout 300 python bench.py --config $cfg --steps 20 --no-cpu-baseline --no-e2e > gpurun_out/ab_t_${cfg}_$tn.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab_t_${cfg}_$tn.json'))
print('$cfg topn=$tn', round(d['value']), [round(v['ms_per_matvec'],4) for v in d['per_nv'].values()], [(round(v['phases_ms']['up_transfer']*1000,1), round(v['phases_ms']['down_transfer']*1000,1)) for v in d['per_nv'].values()])
" >> gpurun_out/ab_topn.txt
  done
done
