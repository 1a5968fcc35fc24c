"""One-line-per-kernel summary of an ncu report (duration, DRAM bytes, occupancy, issue).

    python tools/ncu_brief.py gpurun_out/prof.ncu-rep
"""
import csv
import io
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
           "sm__inst_executed.avg.per_cycle_active", "launch__registers_per_thread",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "lts__t_sectors_srcunit_tex_op_write.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    idx = {m: hdr.index(m) for m in METRICS if m in hdr}
    kn = hdr.index("Kernel Name")
    for r in rows[2:]:
        name = r[kn].split("(")[0]
        parts = [f"{m.split('__')[1].split('.')[0][:18]}={r[i]}{units[i]}" for m, i in idx.items()]
        print(name[:60], "|", " ".join(parts))


if __name__ == "__main__":
    main(sys.argv[1])
