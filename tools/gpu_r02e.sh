set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 2 -c 1 -o gpurun_out/k_step_full -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_density.py -q -x 2>&1 | tail -3
