# rank-order phase 4: phase split, ncu counters against the slot-order build, one full capture
set -x
mkdir -p gpurun_out
MPCD_LIB=build/variants/timing.so timeout 600 python tools/phase_timing.py 256 > gpurun_out/phase_ro.log 2>&1
bash tools/gpu_ncu_ab.sh ro0 ro1 > gpurun_out/ncu_ab_ro.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 2 -c 1 -o gpurun_out/k_step_full_ro -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_ro.log 2>&1
tail -3 gpurun_out/ncu_full_ro.log
