timeout 600 python -m pytest tests/test_gpu_abi.py -q -x 2>&1 | tail -3
