python tools/diag.py --config 5 --reps 3 | grep -v flow
python tools/diag.py --config 3 --reps 3 | grep -v flow
