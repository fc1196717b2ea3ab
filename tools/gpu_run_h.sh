#!/bin/bash
# symmetric-storage and latency-path checks + their bench legs
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/h_build.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests/test_gpu_symmetric.py tests/test_gpu_parity.py -m gpu -q -x -k "symmetric or latency or cfg1 or random" > gpurun_out/h_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/h_pytest.log
timeout 900 python bench.py --config cfg2sym --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/h_cfg2sym.json 2> gpurun_out/h_cfg2sym.err; echo cfg2sym rc=$?
timeout 900 python bench.py --config cfg1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/h_cfg1.json 2> gpurun_out/h_cfg1.err; echo cfg1 rc=$?
H2_MONO=0 timeout 900 python bench.py --config cfg1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/h_cfg1s.json 2> gpurun_out/h_cfg1s.err; echo cfg1s rc=$?
