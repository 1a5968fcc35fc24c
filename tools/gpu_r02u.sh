# both bench arms on one box, final tree
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python bench.py --impl reference > gpurun_out/u_bench_reference.log 2>&1; tail -1 gpurun_out/u_bench_reference.log | cut -c1-400
timeout 900 python bench.py > gpurun_out/u_bench.log 2>&1; tail -1 gpurun_out/u_bench.log | cut -c1-300
