# round-2 re-entry check: full GPU suite, smoke, bench, sanitizer on dense cases
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -40 > gpurun_out/pytest_gpu.log
tail -8 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-1500
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_density.py > gpurun_out/sanitize_memcheck.log 2>&1; tail -8 gpurun_out/sanitize_memcheck.log
timeout 900 python tools/density_sweep.py --out gpurun_out/density_sweep.json > gpurun_out/density_sweep.log 2>&1; tail -8 gpurun_out/density_sweep.log
