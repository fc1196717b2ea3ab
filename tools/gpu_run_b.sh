#!/bin/bash
# round-2 check B: loopback multi-rank parity on one GPU, .h2m on GPU, cfg4 / cfg5 bench legs
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_loopback.py tests/test_h2m_file.py -m gpu -q -rs > gpurun_out/b_pytest.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/b_pytest.log
timeout 900 python bench.py --config cfg4 --steps 10 --warmup 3 > gpurun_out/b_cfg4.json 2> gpurun_out/b_cfg4.err; echo cfg4 rc=$?
timeout 900 python bench.py --config cfg5 --steps 10 --warmup 3 > gpurun_out/b_cfg5.json 2> gpurun_out/b_cfg5.err; echo cfg5 rc=$?
tail -3 gpurun_out/b_cfg5.err
