#!/bin/bash
# latency path: grid size sweep on cfg1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in 8 16 32 64 148; do
H2_MONO_CTAS=$c timeout 300 python bench.py --config cfg1 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/i_cfg1_$c.json 2> gpurun_out/i_cfg1_$c.err; echo $c rc=$?
done
