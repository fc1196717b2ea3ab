#!/bin/bash
# sweep grouping: parity + cfg2 A/B over the group size J
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/k_build.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py -m gpu -q -x > gpurun_out/k_pytest.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/k_pytest.log
for J in 1 2 3 4; do
H2_SWEEP_J=$J timeout 600 python bench.py --config cfg2 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/k_cfg2_$J.json 2> gpurun_out/k_cfg2_$J.err; echo J=$J rc=$?
done
H2_SWEEP_J=3 timeout 600 python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/k_cfg5_3.json 2> gpurun_out/k_cfg5_3.err; echo cfg5 rc=$?
