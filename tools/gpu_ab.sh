set -x
V=build/variants
timeout 900 python tools/ab_time.py $V/base2.so $V/ldg.so --rounds 3 --steps 20 2>&1 | tail -3
