#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
PROF_DTYPE=f32 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_umma --launch-skip 2 --launch-count 1 \
   -o gpurun_out/o_umma python tools/prof_driver.py cfg5 16 > gpurun_out/o_ncu.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/o_ncu.log
