python -m pytest tests -m gpu -x -q 2>&1 | grep -E "Error|error|assert|FAIL|passed|failed" | head -20
python tools/dist_r1_check.py 2>&1 | tail -2
