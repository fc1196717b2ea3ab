#!/bin/bash
# cfg2 per-phase: warp engines vs CTA-tile engine everywhere (nv = 1 and 16)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in "H2_ENGINE=auto" "H2_ENGINE=cta"; do
  env $v timeout 600 python bench.py --steps 10 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/aa.json 2>/dev/null
  echo "$v"; python tools/show.py gpurun_out/aa.json | grep -E "nv=(1|16):" | cut -c1-260
done
