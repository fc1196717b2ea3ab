ARGS="--steps 2 --warmup 3 --no-cpu-baseline --no-e2e --profile-only"
python bench.py $ARGS > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_leaf_dense|k_rows" -s 12 -c 4 \
    -o /tmp/prof_nv16 python bench.py $ARGS > gpurun_out/ncu_nv16.log 2>&1
echo full rc=$?
ncu -i /tmp/prof_nv16.ncu-rep --page raw --csv > gpurun_out/prof_nv16_raw.csv 2>/dev/null
ncu -i /tmp/prof_nv16.ncu-rep --page details --csv > gpurun_out/prof_nv16_details.csv 2>/dev/null
ncu -i /tmp/prof_nv16.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_nv16_source.csv 2>/dev/null
ls -la gpurun_out/prof_nv16*
