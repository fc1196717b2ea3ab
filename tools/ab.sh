timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
for pr in 1 0 1; do H2_PRIO=$pr timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_pr$pr.json 2> gpurun_out/ab_pr$pr.err; echo pr=$pr rc=$?; python -c "
import json; d=json.load(open('gpurun_out/ab_pr$pr.json'))
print('prio $pr', round(d['value']), round(d['ms_per_step'],3), [round(v['ms_per_matvec'],4) for v in d['per_nv'].values()])
"; done
