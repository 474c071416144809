python -m pytest tests -m gpu -x -q 2>&1 | grep -E "Error|error|assert|FAILED|passed|failed|>" | head -30
