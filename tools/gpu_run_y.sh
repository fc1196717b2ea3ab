#!/bin/bash
# sweep grouping A/B on the primary leg (cfg2 nv=1+16)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in "H2_SWEEP_J=4 H2_SWEEP_GMAX=1024" "H2_SWEEP_J=4 H2_SWEEP_GMAX=2048" "H2_SWEEP_J=6 H2_SWEEP_GMAX=1024" "H2_SWEEP_J=8 H2_SWEEP_GMAX=4096" "H2_SWEEP_J=4 H2_SWEEP_GMAX=512"; do
  env $v timeout 600 python bench.py --steps 20 --warmup 5 --no-extra --no-cpu-baseline > gpurun_out/y_ab.json 2>/dev/null
  echo "$v $(python tools/show.py gpurun_out/y_ab.json | grep -E 'nv=(1|16):' | awk '{print $1, $2, $3}' | tr '\n' ' ') $(python tools/show.py gpurun_out/y_ab.json | grep -oE "'up_transfer': [0-9.]+|'down_transfer': [0-9.]+" | tr '\n' ' ')"
done
