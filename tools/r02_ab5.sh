set -x
timeout 1500 python -m pytest tests -x -q -m gpu --timeout 300 2>&1 | tail -3
for ENVS in "X=1" "GAPLA_GROUP_NMAX_THR=32" "GAPLA_GROUP_NMAX_LAT=8" "GAPLA_GROUP_NMAX_LAT=12" "GAPLA_NMAX_NETS_PER_WARP=4"; do
for CFG in 3 5 4; do
  env $ENVS timeout 900 python bench.py --config $CFG --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/b.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b.json'));print('$ENVS cfg$CFG', round(d['value']/1e6,2), 'M nets/s', round(d['ms_per_step'],2), 'ms', round(d['roofline_step']['kernel_ms_per_step']['k_assign'],2))"
done; done
