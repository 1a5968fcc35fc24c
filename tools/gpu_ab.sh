set -x
M=gpu__time_duration.sum,smsp__inst_executed.sum,launch__shared_mem_config_size,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__t_sectors_srcunit_tex_op_atom_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_atom_lookup_hit.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread
MPCD_LIB=build/variants/fz2.so ONLY_WEAK=1 timeout 600 ncu --metrics $M -k regex:k_step -s 30 -c 6 --csv python tools/decomp_overhead.py 192 3 > gpurun_out/ncu_fused.csv 2>&1
grep -E '"(gpu__|smsp|launch|l1tex|lts|dram)' gpurun_out/ncu_fused.csv | awk -F'","' '{print $1, $5, $(NF-2), $NF}' | sed 's/(StepArgs, long)//' | grep -v dense
tail -5 gpurun_out/ncu_fused.csv
