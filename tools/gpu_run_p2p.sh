#!/bin/bash
# device-initiated exchange (NEXT-1) on N GPUs: NCCL-free parity + A/B against the NCCL exchange
N=${1:-2}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_distributed.py -m gpu -q -rs > gpurun_out/x${N}_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/x${N}_pytest.log
for mode in p2p nccl; do
  env H2_EXCHANGE=$mode timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
     --master-port 29543 bench.py --gpus $N --steps 10 --warmup 3 --no-extra > gpurun_out/x${N}_cfg2_$mode.json 2> gpurun_out/x${N}_cfg2_$mode.err
  echo cfg2 $mode rc=$?
  env H2_EXCHANGE=$mode timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
     --master-port 29544 bench.py --gpus $N --steps 10 --warmup 3 --config cfg3 > gpurun_out/x${N}_cfg3_$mode.json 2> gpurun_out/x${N}_cfg3_$mode.err
  echo cfg3 $mode rc=$?
done
