# scratch driver for one-off gpurun diagnostics (edited per experiment), e.g.:
python tools/diag.py --config 5 --reps 3
python tools/diag.py --config 3 --reps 3
