#!/bin/bash
# graph-path A/Bs of the concurrency features (cfg2 primary leg only): default, no PDL, no side stream
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in default H2_PDL=0 H2_SIDE_STREAM=0 "H2_PDL=0 H2_SIDE_STREAM=0"; do
  for rep in 1 2; do
    env $([ "$v" = default ] || echo $v) timeout 600 python bench.py --steps 20 --warmup 5 --no-extra --no-cpu-baseline > gpurun_out/r_ab.json 2>/dev/null
    echo "$v rep$rep $(python tools/show.py gpurun_out/r_ab.json | grep -E 'nv=(1|16):' | awk '{print $1, $2, $3}' | tr '\n' ' ')"
  done
done
