timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python tools/diag.py --config 5 --reps 3 | grep -v flow
python tools/diag.py --config 3 --reps 3
