# ncu of one matvec's k_sweep launches at nv = 16 (DMMA engine), staged vs register-pipelined
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/sw_plain.json 2>/dev/null; echo plain rc=$?
for st in 0 2147483647; do
H2_SSTAGE_MMA=$st timeout 900 ncu --kernel-name regex:k_sweep --launch-skip 30 --launch-count 24 --clock-control none --set full --csv --page raw python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_sweep_$st.csv 2> gpurun_out/ncu_sweep.err; echo ncu rc=$?
done
