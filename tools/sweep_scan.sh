timeout 900 python -m pytest tests/test_samplers_api.py -m gpu -q 2>&1 | tail -3
