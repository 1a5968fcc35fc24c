# round-2 check: density tests, full GPU suite, sanitizer, density sweep, bench
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_density.py -x -q 2>&1 | tail -30 > gpurun_out/pytest_density.log
tail -5 gpurun_out/pytest_density.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_density.py > gpurun_out/sanitize_memcheck.log 2>&1; tail -8 gpurun_out/sanitize_memcheck.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-400
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
timeout 900 python tools/density_sweep.py --out gpurun_out/density_sweep.json > gpurun_out/density_sweep.log 2>&1; tail -3 gpurun_out/density_sweep.log
