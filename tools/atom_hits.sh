# L2 hit/miss of the slot-claim atomics in the steady state (no ncu cache
# flush before the profiled k_step launch), per box edge (GPU box).
cd "$(dirname "$0")/.."
for L in ${@:-256 192}; do
  echo "== L=$L"
  timeout 300 ncu --cache-control none --clock-control none --metrics lts__t_sectors_srcunit_tex_op_atom_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_atom_lookup_miss.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_step -s 4 -c 1 python bench.py --L $L --steps 2 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep -E 'lts__|dram__|gpu__time'
done
