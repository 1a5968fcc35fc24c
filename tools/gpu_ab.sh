set -x
timeout 900 python tools/config5_domain.py 6 2>&1 | tail -9
