timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
H2_MEGA=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
for sp in 1 0; do H2_SPLIT=$sp timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_sp$sp.json 2> gpurun_out/ab_sp$sp.err; echo split=$sp rc=$?; done
