# rank order + unrolled rank groups: GPU tests, bench, launch list, decomposition overhead
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g_pytest_gpu.log 2>&1; tail -2 gpurun_out/g_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.log 2>&1; tail -1 gpurun_out/g_smoke.log
timeout 900 python bench.py > gpurun_out/g_bench.log 2>&1; tail -1 gpurun_out/g_bench.log | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/g_launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/g_b_ncu.log 2>&1
ONLY_WEAK=1 timeout 600 python tools/decomp_overhead.py 224 > gpurun_out/g_decomp.log 2>&1; tail -5 gpurun_out/g_decomp.log
