#!/bin/bash
# pipelined h2_matvec_host: parity + the default bench line's e2e
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "e2e" > gpurun_out/x_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/x_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/x_cfg2.json 2>/dev/null; echo rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/x_cfg2.json').read().strip().splitlines()[-1]); print('value', d['value'], 'e2e', d['e2e'])"
