set -x
MPCD_LIB=build/variants/timing.so timeout 600 python tools/phase_timing.py 256 2>&1 | tail -12
