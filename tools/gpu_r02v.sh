# overflow path out of line (MPCD_OVF_OOL): binned A/B, fused weak form
set -x
mkdir -p gpurun_out
timeout 900 python tools/ab_time.py build/variants/oo0.so build/variants/oo1.so --rounds 4 > gpurun_out/z_ab.log 2>&1
cut -c1-300 gpurun_out/z_ab.log
for v in oo0 oo1; do
  MPCD_LIB=build/variants/$v.so ONLY_WEAK=1 timeout 600 python tools/decomp_overhead.py 224 20 2>&1 | tail -3 | sed "s/^/$v /" >> gpurun_out/z_decomp.log
done
cat gpurun_out/z_decomp.log
