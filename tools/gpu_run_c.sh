#!/bin/bash
# round-2 check C: CTA-tile FP64 engine parity + cfg3 / cfg5 / suite bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/c_build.log 2>&1; echo smoke rc=$?
tail -2 gpurun_out/c_build.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "engines or cfg3 or cfg1 or random" > gpurun_out/c_pytest.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/c_pytest.log
timeout 900 python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c_cfg3.json 2> gpurun_out/c_cfg3.err; echo cfg3 rc=$?
tail -3 gpurun_out/c_cfg3.err
timeout 900 python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c_cfg5.json 2> gpurun_out/c_cfg5.err; echo cfg5 rc=$?
timeout 900 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c_cfg2.json 2> gpurun_out/c_cfg2.err; echo cfg2 rc=$?
H2_ENGINE=warp timeout 900 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c_cfg2w.json 2> gpurun_out/c_cfg2w.err; echo cfg2w rc=$?
