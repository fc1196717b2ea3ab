# final evidence of this build: default bench (cfg2), cfg3s bench, cfg3s launch list, ncu --set full of the cfg3s coupling kernel
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_c.log 2>&1; echo smoke=$? >> gpurun_out/smoke_c.log
timeout 600 python bench.py > gpurun_out/bench_cfg2_c.json 2> gpurun_out/bench_cfg2_c.err
timeout 600 python bench.py --config cfg3s > gpurun_out/bench_cfg3s_c.json 2> gpurun_out/bench_cfg3s_c.err
ARGS="--config cfg3s --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --profile-only"
timeout 300 python bench.py $ARGS > gpurun_out/plain_c.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/launches_cfg3s_c.csv python bench.py $ARGS > gpurun_out/ncu_launch_c.log 2>&1
echo launches rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_rows|k_leaf_dense_split|k_sweep" -s 30 -c 4 \
    -o /tmp/prof_c python bench.py $ARGS > gpurun_out/ncu_full_c.log 2>&1
echo full rc=$?
ncu -i /tmp/prof_c.ncu-rep --page raw --csv > gpurun_out/prof_c_raw.csv 2>/dev/null
ncu -i /tmp/prof_c.ncu-rep --page details --csv > gpurun_out/prof_c_details.csv 2>/dev/null
ls -la gpurun_out/
