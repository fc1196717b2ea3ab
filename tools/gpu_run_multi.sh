#!/bin/bash
# multi-GPU evidence on N GPUs of one box: NCCL parity (tests/test_gpu_distributed.py via torchrun)
# and the default bench line (cfg2 weak + cfg3 strong + cfg1) plus cfg5 / cfg4 weak scaling.
N=${1:-2}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_distributed.py -m gpu -q -rs > gpurun_out/m${N}_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/m${N}_pytest.log
for cfg in ${CFGS:-suite cfg5 cfg4}; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29541 \
     bench.py --gpus $N --steps 10 --warmup 3 --config $cfg > gpurun_out/m${N}_$cfg.json 2> gpurun_out/m${N}_$cfg.err
  echo $cfg rc=$?
done
