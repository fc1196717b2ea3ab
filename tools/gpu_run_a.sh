#!/bin/bash
# round-2 check A: stripped library GPU suite + full-size parity + default suite bench
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/a_smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/a_pytest.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/a_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/a_bench.json 2> gpurun_out/a_bench.err; echo bench rc=$?
tail -3 gpurun_out/a_bench.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/a_ref.json 2> gpurun_out/a_ref.err; echo ref rc=$?
