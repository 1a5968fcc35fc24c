# staging columns as the default (non-fused modes): GPU tests, smoke, bench, launch list
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/n_pytest_gpu.log 2>&1; tail -2 gpurun_out/n_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/n_smoke.log 2>&1; tail -1 gpurun_out/n_smoke.log
timeout 900 python bench.py > gpurun_out/n_bench.log 2>&1; tail -1 gpurun_out/n_bench.log | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/n_launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/n_b_ncu.log 2>&1
