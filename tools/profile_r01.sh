# ncu evidence for round 1 (B200_PROFILING.md recipe); run under gpurun on 1 GPU.
# Exports CSV summaries on the box (the .ncu-rep itself is too large to bring back).
ARGS="--steps 2 --warmup 3 --no-cpu-baseline --no-e2e --profile-only"
python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/launches_r01.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1
echo launches rc=$?
python bench.py $ARGS > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_dense|k_rows|k_leaf_u|k_up_leaf" -s 40 -c 6 \
    -o /tmp/prof_r01 python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1
echo full rc=$?
ncu -i /tmp/prof_r01.ncu-rep --page raw --csv > gpurun_out/prof_r01_raw.csv 2>/dev/null
ncu -i /tmp/prof_r01.ncu-rep --page details --csv > gpurun_out/prof_r01_details.csv 2>/dev/null
ls -la gpurun_out/
