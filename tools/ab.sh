timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
for st in 1 0; do H2_SUBTREE=$st timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_st$st.json 2> gpurun_out/ab_st$st.err; echo st=$st rc=$?; done
