#!/bin/bash
# final ncu full sets: symmetric kernels (cfg2:sym) and the tcgen05 FP32 kernels (cfg5 f32)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sym --launch-skip 4 --launch-count 2 \
   -o gpurun_out/fin_sym python bench.py --config cfg2sym --steps 1 --warmup 1 --profile-only --no-cpu-baseline > gpurun_out/fin_ncu1.log 2>&1; echo ncu1 rc=$?
PROF_DTYPE=f32 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_umma --launch-skip 3 --launch-count 2 \
   -o gpurun_out/fin_umma python tools/prof_driver.py cfg5 16 > gpurun_out/fin_ncu2.log 2>&1; echo ncu2 rc=$?
