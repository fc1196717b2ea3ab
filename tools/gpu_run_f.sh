#!/bin/bash
# FD solve (NEXT-4) on the GPU + full GPU suite
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f_build.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -q -x -rs > gpurun_out/f_pytest.log 2>&1; echo pytest rc=$?
tail -4 gpurun_out/f_pytest.log
