GAPLA_SLOT_BYTES=2816 python tools/diag.py --config 5 --reps 3 | grep -v flow
GAPLA_SLOT_BYTES=3328 python tools/diag.py --config 5 --reps 3 | grep -v flow
python tools/diag.py --config 5 --reps 3 | grep -v flow
