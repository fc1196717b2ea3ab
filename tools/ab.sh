timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_split_tu.json 2> gpurun_out/bench_split_tu.err; echo rc=$?
