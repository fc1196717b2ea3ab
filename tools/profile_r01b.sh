# Round-1 evidence (final state): bench line, reference arm, launch list, full-set capture of the top kernels
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r01b.json 2> gpurun_out/bench_r01b.err; echo bench rc=$?
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_r01.json 2> gpurun_out/bench_ref_r01.err; echo ref rc=$?
ARGS="--steps 2 --warmup 3 --no-cpu-baseline --no-e2e --profile-only"
python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/launches_r01b.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1
echo launches rc=$?
python bench.py $ARGS > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_leaf_dense|k_rows|k_up_leaf|k_sweep" -s 0 -c 40 \
    -o /tmp/prof_r01b python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1
echo full rc=$?
ncu -i /tmp/prof_r01b.ncu-rep --page raw --csv > gpurun_out/prof_r01b_raw.csv 2>/dev/null
ls -la gpurun_out/*r01b*
