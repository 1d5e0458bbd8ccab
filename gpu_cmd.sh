timeout 900 python -m pytest tests -m gpu -q -rf -x 2>&1 | tail -12
