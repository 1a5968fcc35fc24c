#!/bin/bash
# Run the bench once per tuning variant in build/variants (GPU box).
cd "$(dirname "$0")/.."
for so in build/variants/*.so; do
  name=$(basename "$so" .so)
  line=$(MPCD_LIB="$so" timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1)
  python - "$name" "$line" <<'PY'
import json, sys
name, line = sys.argv[1], sys.argv[2]
try:
    d = json.loads(line)
    print(f"{name:12s} ms/step {d['ms_per_step']:.3f}  Gps {d['value']/1e9:.2f}  k_step {d['roofline_step']['kernel_ms']['k_step']:.3f}")
except Exception:
    print(name, "FAILED", line[-300:])
PY
done
