#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sym --launch-skip 4 --launch-count 2 \
   -o gpurun_out/u_sym python bench.py --config cfg2sym --steps 1 --warmup 1 --profile-only --no-cpu-baseline > gpurun_out/u_ncu.log 2>&1; echo ncu rc=$?
tail -2 gpurun_out/u_ncu.log
