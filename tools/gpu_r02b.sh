nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
V=build/variants
timeout 600 python tools/ab_time.py $V/r01_head.so $V/cur3.so $V/tc32f16.so --rounds 3 --steps 20 2>&1 | tail -3
timeout 300 python tools/ab_time.py $V/r01_head.so $V/cur3.so --density 4 --rounds 1 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_density.py -x -q 2>&1 | tail -30 > gpurun_out/pytest_density.log; tail -3 gpurun_out/pytest_density.log
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -40 > gpurun_out/pytest_gpu.log; tail -8 gpurun_out/pytest_gpu.log
