#!/bin/bash
# symmetric kernels: parity + cfg2sym / cfg4sym legs
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_symmetric.py -m gpu -q -x > gpurun_out/v_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/v_pytest.log
for c in cfg2sym cfg4sym; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/v_$c.json 2>/dev/null; echo $c rc=$?
  python tools/show.py gpurun_out/v_$c.json | head -3
done
