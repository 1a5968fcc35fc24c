# early release as the default: GPU tests, smoke, bench, launch list, ncu brief, fused weak form
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/t_pytest_gpu.log 2>&1; tail -2 gpurun_out/t_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t_smoke.log 2>&1; tail -1 gpurun_out/t_smoke.log
timeout 900 python bench.py > gpurun_out/t_bench.log 2>&1; tail -1 gpurun_out/t_bench.log | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/t_launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/t_b_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 2 -c 1 -o gpurun_out/k_step_full_t -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/t_ncu_full.log 2>&1
ONLY_WEAK=1 timeout 600 python tools/decomp_overhead.py 224 20 > gpurun_out/t_decomp.log 2>&1; tail -3 gpurun_out/t_decomp.log
