timeout 900 python -m pytest tests/test_gpu_distributed.py -m gpu -q -x -s 2>&1 | grep -E "dist P=|passed|failed" | tail -14
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_p4.json 2> gpurun_out/bench_p4.err; echo p4 rc=$?
