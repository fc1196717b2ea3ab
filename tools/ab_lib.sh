# A/B of prebuilt library variants paper_2109_05451_b200/var_*.so (bench only)
L=paper_2109_05451_b200/libh2b200.so
for rep in 1 2; do for v in "$@"; do
  cp paper_2109_05451_b200/var_$v.so $L
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ablib.json 2> gpurun_out/ablib.err || echo "rc=$? $v"
  python -c "
import json; d=json.load(open('gpurun_out/ablib.json'))
print('$v', round(d['value']), [round(v['ms_per_matvec'],4) for v in d['per_nv'].values()], {k: round(x*1000,1) for k,x in d['per_nv']['16']['phases_ms'].items() if x>0.01})
"; done; done
