#!/bin/bash
# Run the bench (and a quick parity subset) once per tuning variant in
# build/variants (GPU box).  MPCD_LIB selects the library (paper_2212_11878_b200/_lib.py).
cd "$(dirname "$0")/.."
for so in build/variants/*.so; do
  name=$(basename "$so" .so)
  par=$(MPCD_LIB="$so" timeout 300 python -m pytest tests/test_gpu_parity.py -q -x \
        -k "64cubed or config1 or dense or conservation" 2>&1 | tail -1)
  line=$(MPCD_LIB="$so" timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1)
  python - "$name" "$line" "$par" <<'PY'
import json, sys
name, line, par = sys.argv[1], sys.argv[2], sys.argv[3]
try:
    d = json.loads(line)
    k = d['roofline_step']['kernel_ms']
    print(f"{name:12s} ms/step {d['ms_per_step']:.3f}  Gps {d['value']/1e9:.2f}  k_step {k['k_step']:.3f} dense {k['k_step_dense']:.3f} | {par}")
except Exception:
    print(name, "FAILED", line[-300:], par)
PY
done
