"""Executed warp-instructions of one kernel per CUDA source line, from an ncu
report (SASS page) joined with the line table of the in-tree library
(nvdisasm --print-line-info), plus a per-phase total for k_step's consumer
phases (the "// phase N" comments of mpcd_step.cuh).

    python tools/ncu_lines.py gpurun_out/k_step_full.ncu-rep [mangled-kernel-name] [top]
"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2212_11878_b200", "libmpcd.so")
STEP = os.path.join(ROOT, "paper_2212_11878_b200", "csrc", "mpcd_step.cuh")


def sass_counts(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    kern = rows[0][1] if rows and rows[0] and rows[0][0] == "Kernel Name" else ""
    hdr = rows[1]
    ia, ie = hdr.index("Address"), hdr.index("Instructions Executed")
    data = []
    for r in rows[2:]:
        if len(r) <= ie:
            continue
        try:
            data.append((int(r[ia], 16), float(r[ie] or 0)))
        except ValueError:
            continue
    return kern, data


def line_table(mangled):
    with tempfile.TemporaryDirectory() as tmp:
        subprocess.run(["cuobjdump", "-xelf", "all", LIB], cwd=tmp, capture_output=True)
        for f in sorted(os.listdir(tmp)):
            if not f.endswith(".cubin"):
                continue
            txt = subprocess.run(["nvdisasm", "--print-line-info", os.path.join(tmp, f)],
                                 capture_output=True, text=True).stdout
            sec = re.search(r"\.text\." + re.escape(mangled) + r" -+\n(.*?)(?:\n//-+ \.text|\Z)",
                            txt, re.S)
            if not sec:
                continue
            cur, table = None, {}
            for line in sec.group(1).splitlines():
                m = re.search(r'## File "([^"]+)", line (\d+)', line)
                if m:
                    cur = (os.path.basename(m.group(1)), int(m.group(2)))
                    continue
                m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", line)
                if m:
                    table[int(m.group(1), 16)] = cur
            return table
    return {}


def phases():
    """(line, name) markers of consume_cells' phases in mpcd_step.cuh."""
    marks = []
    for i, line in enumerate(open(STEP), 1):
        m = re.match(r"\s*// phase (\d)", line)
        if m:
            marks.append((i, f"phase {m.group(1)}"))
    return marks


def main(rep, mangled="_ZN4mpcd6k_stepILb1ELb1ELb0ELb0ELi0ELi16EEEvNS_8StepArgsEl", top=30):
    """mangled: the profiled kernel's symbol (default: the binned unit-mass
    16-cell variant the bench runs)."""
    kern, data = sass_counts(rep)
    table = line_table(mangled) if mangled else {}
    base = min(a for a, _ in data)
    per_line = defaultdict(float)
    for a, e in data:
        per_line[table.get(a - base)] += e
    tot = sum(per_line.values())
    src = open(STEP).read().splitlines()
    print(f"{kern[:70]}: {tot:.3e} warp-instructions")
    for (key, e) in sorted(per_line.items(), key=lambda kv: -kv[1])[:top]:
        text = ""
        if key and key[0] == "mpcd_step.cuh":
            text = src[key[1] - 1].strip()[:70]
        print(f"{e / tot * 100:5.1f}%  {str(key):28s} {text}")
    marks = phases()
    if marks:
        buckets = defaultdict(float)
        for key, e in per_line.items():
            name = "other"
            if key and key[0] == "mpcd_step.cuh":
                for ln, nm in marks:
                    if key[1] >= ln:
                        name = nm
            buckets[name] += e
        print("--- by phase marker (lines after '// phase N' up to the next marker)")
        for k, v in sorted(buckets.items()):
            print(f"  {k:10s} {v / tot * 100:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], *(sys.argv[2:3] or []), *(int(x) for x in sys.argv[3:4]))
