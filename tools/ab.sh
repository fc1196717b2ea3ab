# A/B: parity + two bench repetitions of the current build (tag $1)
tag=${1:-cur}
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -25
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err; echo rc=$?; python -c "
import json; d=json.load(open('gpurun_out/ab_$tag.json'))
print('$tag', round(d['value']), round(d['ms_per_step'],3), [round(v['ms_per_matvec'],4) for v in d['per_nv'].values()])
for k,v in d['per_nv'].items(): print(k, {a: round(x*1000,1) for a,x in v['phases_ms'].items()})
"; done
