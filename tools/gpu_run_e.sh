#!/bin/bash
# CTA engine warp-tile variants on cfg3 (nv=64)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in 0 1 2; do
H2_CTA_VAR=$v timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "engines" > gpurun_out/e_pytest$v.log 2>&1; echo pytest$v rc=$?
H2_CTA_VAR=$v timeout 900 python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/e_cfg3_$v.json 2> gpurun_out/e_cfg3_$v.err; echo cfg3 $v rc=$?
done
