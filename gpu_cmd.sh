timeout 900 python -m pytest tests/test_gpu_pool.py -q -x 2>&1 | tail -8
