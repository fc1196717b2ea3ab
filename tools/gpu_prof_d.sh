#!/bin/bash
# ncu full-set captures of the CTA engine (coupling launch) at nv=16 and nv=64 on cfg3s
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
H2_ENGINE=cta timeout 300 python tools/prof_driver.py cfg3s 16 64 > gpurun_out/d_plain.log 2>&1; echo plain rc=$?
H2_ENGINE=cta timeout 900 ncu --set full --import-source on -k regex:k_cta --launch-skip 1 --launch-count 1 \
   -o gpurun_out/d_cta16 python tools/prof_driver.py cfg3s 16 > gpurun_out/d_ncu16.log 2>&1; echo ncu16 rc=$?
H2_ENGINE=cta timeout 900 ncu --set full --import-source on -k regex:k_cta --launch-skip 1 --launch-count 1 \
   -o gpurun_out/d_cta64 python tools/prof_driver.py cfg3s 64 > gpurun_out/d_ncu64.log 2>&1; echo ncu64 rc=$?


