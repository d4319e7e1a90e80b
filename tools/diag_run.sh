timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
GAPLA_VERBOSE=1 python tools/e2e_diag.py --config 5 2>&1 | grep -E "rep|upload|GPU batching"
