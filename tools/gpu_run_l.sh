#!/bin/bash
# FP32 tensor engine: parity (incl. cfg5 full size) + cfg5 bench; p2p early leaf off-diagonal check at P=1 paths
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/l_build.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_loopback.py -m gpu -q -x -k "fp32 or f32 or engines or cfg1 or random" > gpurun_out/l_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/l_pytest.log
timeout 900 python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/l_cfg5.json 2> gpurun_out/l_cfg5.err; echo cfg5 rc=$?
