set -x
V=build/variants
timeout 900 python tools/ab_time.py $V/prod3.so $V/ob.so --rounds 3 --steps 20 2>&1 | tail -4
