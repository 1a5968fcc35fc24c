# fused (decomposed) k_step against the whole-box k_step: one full capture each, 224^3 weak form
set -x
mkdir -p gpurun_out
export ONLY_WEAK=1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:'k_stepILb1ELb1ELb0ELb0ELi3ELi16' -s 2 -c 1 -o gpurun_out/k_step_fused_full -f python tools/decomp_overhead.py 224 3 > gpurun_out/h_ncu_fused.log 2>&1
tail -2 gpurun_out/h_ncu_fused.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:'k_stepILb1ELb1ELb0ELb0ELi0ELi16' -s 2 -c 1 -o gpurun_out/k_step_whole224_full -f python tools/decomp_overhead.py 224 3 > gpurun_out/h_ncu_whole.log 2>&1
tail -2 gpurun_out/h_ncu_whole.log
