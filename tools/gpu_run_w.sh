#!/bin/bash
# cfg2 primary leg A/B for a leaf-kernel variant (parity of the DMMA leaf first)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "cfg2 or random or engines" > gpurun_out/w_pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/w_pytest.log
for rep in 1 2; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-extra --no-cpu-baseline > gpurun_out/w_cfg2.json 2>/dev/null; echo rc=$?
python tools/show.py gpurun_out/w_cfg2.json | grep -E "nv=" | cut -c1-200
done
