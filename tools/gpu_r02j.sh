# fused leavers out of line as the default: GPU tests, decomposition overhead
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/j_pytest_gpu.log 2>&1; tail -2 gpurun_out/j_pytest_gpu.log
ONLY_WEAK=1 timeout 600 python tools/decomp_overhead.py 224 20 > gpurun_out/j_decomp.log 2>&1; tail -3 gpurun_out/j_decomp.log
timeout 600 python tools/decomp_overhead.py 256 10 > gpurun_out/j_decomp256.log 2>&1; tail -12 gpurun_out/j_decomp256.log
