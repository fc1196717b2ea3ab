# cfg3s evidence (compute-bound nv=64 regime): parity, bench line, ncu launch list; 1 GPU under gpurun.
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "cfg3" > gpurun_out/pytest_cfg3.log 2>&1
echo pytest=$? >> gpurun_out/pytest_cfg3.log
timeout 600 python bench.py --config cfg3s > gpurun_out/bench_cfg3s.json 2> gpurun_out/bench_cfg3s.err
echo bench rc=$?
ARGS="--config cfg3s --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --profile-only"
timeout 300 python bench.py $ARGS > gpurun_out/plain_cfg3s.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/launches_cfg3s.csv python bench.py $ARGS > gpurun_out/ncu_launch_cfg3s.log 2>&1
echo launches rc=$?
