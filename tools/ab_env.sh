# A/B of env settings: tools/ab_env.sh "NAME=V1" "NAME=V2" ...  (parity first, default env)
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -25
for rep in 1 2; do for cfg in "$@"; do
  env $cfg timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/abenv.json 2> gpurun_out/abenv.err || echo "rc=$? $cfg"
  python -c "
import json; d=json.load(open('gpurun_out/abenv.json'))
print('$cfg', round(d['value']), [round(v['ms_per_matvec'],4) for v in d['per_nv'].values()], [(round(v['phases_ms']['up_transfer']*1000,1), round(v['phases_ms']['down_transfer']*1000,1)) for v in d['per_nv'].values()])
"; done; done
