timeout 900 python -m pytest tests/test_gpu_distributed.py -m gpu -q -x 2>&1 | tail -4
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_p2.json 2> gpurun_out/bench_p2.err; echo p2 rc=$?
