set -x
timeout 1200 python -m pytest tests/test_gpu_distributed.py -q -x 2>&1 | tail -3
