set -x
timeout 900 python tools/pcie_probe.py 2>&1 | tail -8
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_density.py -q -x 2>&1 | tail -3
