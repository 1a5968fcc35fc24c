"""Summarise an `ncu --page source --print-source sass --csv` export:
instructions executed and stall samples per opcode, and the hottest lines.

    ncu -i rep.ncu-rep --page source --csv --kernel-name K --print-source sass > k.csv
    python tools/ncu_sass_summary.py k.csv
"""
import csv
import sys
from collections import defaultdict


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ia, isrc = hdr.index("Address"), hdr.index("Source")
    iex = hdr.index("Instructions Executed")
    ist = hdr.index("Warp Stall Sampling (All Samples)")
    by_op = defaultdict(lambda: [0, 0, 0])
    lines = []
    for r in rows[2:]:
        if len(r) <= max(ist, iex):
            continue
        op = r[isrc].split()[0] if r[isrc].split() else "?"
        if op.startswith("@"):
            op = r[isrc].split()[1]
        try:
            ex = float(r[iex] or 0)
            st = float(r[ist] or 0)
        except ValueError:  # repeated header of the next launch
            continue
        by_op[op][0] += ex
        by_op[op][1] += st
        by_op[op][2] += 1
        lines.append((st, ex, r[ia], r[isrc]))
    tot_ex = sum(v[0] for v in by_op.values())
    tot_st = sum(v[1] for v in by_op.values())
    print(f"static instructions {len(lines)}, executed {tot_ex:.3e}, stall samples {tot_st:.0f}")
    for op, (ex, st, cnt) in sorted(by_op.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{op:28s} exec {ex / tot_ex * 100:5.1f}%  stall {st / max(tot_st, 1) * 100:5.1f}%  static {cnt}")
    print("--- hottest instructions by stall samples")
    for st, ex, a, s in sorted(lines, reverse=True)[:top]:
        print(f"{st:8.0f} {ex:12.0f} {a} {s[:90]}")




def lines_main(path, top=30):
    """Per-CUDA-line view of an `--print-source cuda,sass --csv` export."""
    rows = list(csv.reader(open(path)))
    seen = {}
    for r in rows:
        if len(r) > 8 and r[0].isdigit():
            try:
                seen[int(r[0])] = (float(r[4] or 0), float(r[7] or 0), r[1])
            except ValueError:
                pass
    tot_st = sum(v[0] for v in seen.values()) or 1
    tot_ex = sum(v[1] for v in seen.values()) or 1
    print(f"lines {len(seen)}  stall samples {tot_st:.0f}  warp-instructions {tot_ex:.3e}")
    print("--- by stall samples")
    for ln, (st, ex, src) in sorted(seen.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{ln:5d} stall {st / tot_st * 100:5.1f}%  inst {ex / tot_ex * 100:5.1f}%  {src.strip()[:80]}")
    print("--- by instructions executed")
    for ln, (st, ex, src) in sorted(seen.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{ln:5d} inst {ex / tot_ex * 100:5.1f}%  stall {st / tot_st * 100:5.1f}%  {src.strip()[:80]}")


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[2] == "lines":
        lines_main(sys.argv[1])
    else:
        main(sys.argv[1])
