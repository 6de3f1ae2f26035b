timeout 900 python -m pytest tests/ -q -m "gpu" --timeout=180 2>&1 | grep -E "passed|failed|error|FAIL" | tail -15
