#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
H2_DEBUG=1 H2_EXCHANGE=p2p timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29547 tests/dist_worker.py > gpurun_out/dbg_p2p.log 2>&1; echo rc=$?
grep -E "h2 error|rel err|FAIL|OK|stuck|p2p" gpurun_out/dbg_p2p.log | head -20
