#!/bin/bash
# round-2 final-ish: full single-GPU suite + the default bench line + cfg5 / cfg4 / cfg4sym legs
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/q_build.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -q -x -rs > gpurun_out/q_pytest.log 2>&1; echo pytest rc=$?
tail -4 gpurun_out/q_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/q_suite.json 2> gpurun_out/q_suite.err; echo suite rc=$?
for c in cfg5 cfg4 cfg4sym cfg2sym; do
timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/q_$c.json 2> gpurun_out/q_$c.err; echo $c rc=$?
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/q_ref.json 2> gpurun_out/q_ref.err; echo ref rc=$?
