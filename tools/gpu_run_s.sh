#!/bin/bash
# default bench line (suite incl. the cfg5 FP32 tcgen05 leg) with its wall time; smoke
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s_build.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/s_build.log
t0=$(date +%s); timeout 1200 python bench.py > gpurun_out/s_suite.json 2> gpurun_out/s_suite.err; echo suite rc=$? wall=$(( $(date +%s) - t0 ))s
python tools/show.py gpurun_out/s_suite.json
