timeout 600 python -m pytest tests/test_decode_gpu.py -x -q 2>&1 | grep -E "Error|error|assert|FAILED|passed|failed" | head -20
