python tools/diag.py --config 5 --reps 2
python tools/diag.py --config 3 --reps 2
