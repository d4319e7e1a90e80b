GAPLA_WARP_BIG=1 timeout 900 python -m pytest tests -x -q -m gpu -k "config or dense or snapshot" 2>&1 | tail -2
python tools/diag.py --config 5 --reps 2 | grep -v flow
GAPLA_WARP_BIG=1 python tools/diag.py --config 5 --reps 2 | grep -v flow
GAPLA_WARP_BIG=1 python tools/diag.py --config 3 --reps 2 | grep -v flow
