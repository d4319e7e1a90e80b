timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 900 python bench.py --config 1 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('cfg1', d['value']/1e6, d['ms_per_step'])"
