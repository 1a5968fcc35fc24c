nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
V=build/variants
timeout 600 python tools/ab_time.py $V/r01_head.so $V/cur.so $V/cur.so:MPCD_BRICK=1 $V/tc32.so --rounds 3 --steps 20 2>&1 | tail -5
timeout 300 python tools/ab_time.py $V/cur.so $V/tc32.so --density 4 --rounds 2 2>&1 | tail -3
timeout 300 python tools/ab_time.py $V/cur.so $V/tc32.so --density 6 --rounds 2 2>&1 | tail -3
timeout 300 python tools/ab_time.py $V/cur.so $V/cur.so:MPCD_BRICK=1 --density 15 --L 192 --rounds 2 2>&1 | tail -3
