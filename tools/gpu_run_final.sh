#!/bin/bash
# final check: build + smoke, full single-GPU test suite, default bench line
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f_build.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/f_build.log
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/f_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/f_pytest.log
timeout 900 python bench.py > gpurun_out/f_suite.json 2> gpurun_out/f_suite.err; echo suite rc=$?
