nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
V=build/variants
timeout 900 python tools/ab_time.py $V/r01_head.so $V/cur2.so $V/fixed16.so $V/tc32.so $V/tc32f16.so --rounds 3 --steps 20 2>&1 | tail -6
