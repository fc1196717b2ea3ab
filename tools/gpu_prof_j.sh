#!/bin/bash
# round-2 ncu evidence: launch list of the default bench line, full-set captures of the dominant kernels
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/j_launches.csv python bench.py --steps 2 --warmup 3 --profile-only > gpurun_out/j_launch.log 2>&1; echo launches rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_leaf_dense --launch-count 2 \
   -o gpurun_out/j_cfg2_leaf python tools/prof_driver.py cfg2 1 16 > gpurun_out/j_ncu1.log 2>&1; echo ncu_cfg2 rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_cta --launch-skip 1 --launch-count 1 \
   -o gpurun_out/j_cfg3_coup python tools/prof_driver.py cfg3 64 > gpurun_out/j_ncu2.log 2>&1; echo ncu_cfg3c rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_cta --launch-skip 32 --launch-count 1 \
   -o gpurun_out/j_cfg3_leaf python tools/prof_driver.py cfg3 64 > gpurun_out/j_ncu3.log 2>&1; echo ncu_cfg3l rc=$?
