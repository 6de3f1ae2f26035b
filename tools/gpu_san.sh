timeout 900 python -m pytest tests/ -q -m "gpu" --timeout=300 2>&1 | grep -E "passed|failed|error|FAIL" | tail -15
for tool in memcheck racecheck synccheck; do
  echo "== $tool"; timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_run.py 2>&1 | tail -4
done
