#!/bin/bash
# nv=16 evidence: full sets of the cfg2 leaf kernel and coupling at nv=16 (FP64 DMMA) and cfg5 FP32 coupling (3xTF32)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -o gpurun_out/umma_probe tools/umma_probe.cu > gpurun_out/n_probe.log 2>&1; timeout 60 gpurun_out/umma_probe >> gpurun_out/n_probe.log 2>&1; echo probe rc=$?; cat gpurun_out/n_probe.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_leaf_dense --launch-skip 1 --launch-count 1 \
   -o gpurun_out/n_cfg2_leaf16 python tools/prof_driver.py cfg2 16 > gpurun_out/n_ncu1.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_rows --launch-skip 2 --launch-count 2 \
   -o gpurun_out/n_cfg2_rows16 python tools/prof_driver.py cfg2 16 > gpurun_out/n_ncu2.log 2>&1; echo ncu2 rc=$?
PROF_DTYPE=f32 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_rows --launch-skip 2 --launch-count 2 \
   -o gpurun_out/n_cfg5_rows_f32 python tools/prof_driver.py cfg5 16 > gpurun_out/n_ncu3.log 2>&1; echo ncu3 rc=$?
nvcc -gencode arch=compute_100a,code=sm_100a -o gpurun_out/umma_probe tools/umma_probe.cu > gpurun_out/n_probe.log 2>&1
timeout 60 gpurun_out/umma_probe >> gpurun_out/n_probe.log 2>&1; echo probe rc=$?
cat gpurun_out/n_probe.log
