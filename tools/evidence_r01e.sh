# final evidence (2-GPU box): full GPU suite incl. P=2 parity, then 1-GPU bench lines (cfg2 default, cfg3s)
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_e.log 2>&1; echo pytest=$? >> gpurun_out/pytest_e.log
export CUDA_VISIBLE_DEVICES=0
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_e.log 2>&1; echo smoke=$? >> gpurun_out/smoke_e.log
timeout 600 python bench.py > gpurun_out/bench_cfg2_e.json 2> gpurun_out/bench_cfg2_e.err
timeout 600 python bench.py --config cfg3s > gpurun_out/bench_cfg3s_e.json 2> gpurun_out/bench_cfg3s_e.err
timeout 600 python bench.py --impl reference --config cfg3s --steps 1 > gpurun_out/bench_cfg3s_ref_e.json 2> gpurun_out/bench_cfg3s_ref_e.err
ls -la gpurun_out
