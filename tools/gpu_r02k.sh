# flat phase 2 / hoisted cache policy: binned A/B and the fused weak form
set -x
mkdir -p gpurun_out
timeout 900 python tools/ab_time.py build/variants/pf0.so build/variants/pf1.so build/variants/pn1.so build/variants/pfn1.so --rounds 4 > gpurun_out/k_ab.log 2>&1
cut -c1-300 gpurun_out/k_ab.log
for v in pf0 pn1; do
  MPCD_LIB=build/variants/$v.so ONLY_WEAK=1 timeout 600 python tools/decomp_overhead.py 224 20 2>&1 | tail -3 | sed "s/^/$v /" >> gpurun_out/k_decomp.log
done
cat gpurun_out/k_decomp.log
