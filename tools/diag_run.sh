timeout 1200 python -m pytest tests -x -q -m gpu -k "config or snapshot or dense" 2>&1 | tail -2
GAPLA_VERBOSE=1 python tools/e2e_diag.py --config 5 2>&1 | grep -E "rep|priority"
