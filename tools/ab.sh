timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
for cfg in "0 2" "1 2" "1 1"; do set -- $cfg
  H2_CHAIN=$1 H2_CHAIN_CTAS=$2 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_c$1_$2.json 2> gpurun_out/ab_c$1_$2.err; echo chain=$1 ctas=$2 rc=$?; done
