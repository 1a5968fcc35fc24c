# ncu counters of k_step for several variant builds (one launch each)
set -x
mkdir -p gpurun_out
M=gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__inst_executed.sum,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_atom_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_atom_lookup_miss.sum
for v in "$@"; do
  timeout 300 ncu --metrics $M --clock-control none -k regex:k_step -s 4 -c 1 --csv python tools/ab_time.py build/variants/$v.so --rounds 1 --steps 3 --hash 0 --split 0 > gpurun_out/ncu_ab_$v.csv 2>&1
  grep -E '"(gpu__time|l1tex|smsp|dram|lts)' gpurun_out/ncu_ab_$v.csv | awk -F'","' -v v=$v '{print v, $(NF-2), $NF}'
done
