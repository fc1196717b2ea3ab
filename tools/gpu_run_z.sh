#!/bin/bash
# cfg3 (nv = 64): CTA-tile transfer levels vs warp sweeps
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in "H2_CTA_SWEEPS=1" "H2_CTA_SWEEPS=0"; do
  env $v timeout 900 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/z_ab.json 2>/dev/null
  echo "$v $(python tools/show.py gpurun_out/z_ab.json | grep -E 'nv=64:' | cut -c1-230)"
done
H2_CTA_SWEEPS=0 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "cfg3 or engines" > gpurun_out/z_pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/z_pytest.log
