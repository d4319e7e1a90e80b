timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python tools/diag.py --config 3 --reps 2
python tools/diag.py --config 5 --reps 2
