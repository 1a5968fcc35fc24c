# final evidence of the late round-2 kernel: GPU tests, smoke, bench, launch list, ncu brief, memcheck
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/l_pytest_gpu.log 2>&1; tail -2 gpurun_out/l_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/l_smoke.log 2>&1; tail -1 gpurun_out/l_smoke.log
timeout 900 python bench.py > gpurun_out/l_bench.log 2>&1; tail -1 gpurun_out/l_bench.log | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/l_launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/l_b_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 2 -c 1 -o gpurun_out/k_step_full_final -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/l_ncu_full.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_density.py > gpurun_out/l_sanitize_memcheck.log 2>&1; tail -3 gpurun_out/l_sanitize_memcheck.log
ONLY_WEAK=1 timeout 600 python tools/decomp_overhead.py 224 20 > gpurun_out/l_decomp.log 2>&1; tail -3 gpurun_out/l_decomp.log
