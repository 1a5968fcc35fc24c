# fused leavers out of line: decomposition overhead per build (224^3 weak form)
set -x
mkdir -p gpurun_out
for v in fo0 fo1 fo0 fo1; do
  MPCD_LIB=build/variants/$v.so ONLY_WEAK=1 timeout 600 python tools/decomp_overhead.py 224 20 2>&1 | tail -3 | sed "s/^/$v /" >> gpurun_out/i_decomp.log
done
cat gpurun_out/i_decomp.log
