#!/bin/bash
# tcgen05 FP32 coupling engine: parity first (bounded), then cfg5 f32 bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/o_build.log 2>&1; echo build rc=$?
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py -m gpu -q -x -k "fp32" > gpurun_out/o_pytest.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/o_pytest.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -k "f32" > gpurun_out/o_pytest2.log 2>&1; echo pytest2 rc=$?
tail -3 gpurun_out/o_pytest2.log
timeout 600 python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/o_cfg5.json 2> gpurun_out/o_cfg5.err; echo cfg5 rc=$?
python tools/show.py gpurun_out/o_cfg5.json
PROF_DTYPE=f32 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_umma --launch-skip 3 --launch-count 2 \
   -o gpurun_out/o_umma python tools/prof_driver.py cfg5 16 > gpurun_out/o_ncu.log 2>&1; echo ncu rc=$?
