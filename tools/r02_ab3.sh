# quick benches of alternate builds (GAPLA_SO), no parity
for SO in ${SOS:-libgapla.so}; do
for CFG in ${CFGS:-3 5}; do
  GAPLA_SO=$SO timeout 900 python bench.py --config $CFG --no-e2e --no-cpu-baseline --steps ${STEPS:-10} > gpurun_out/b_${SO}_$CFG.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b_${SO}_$CFG.json'));print('$SO cfg$CFG', round(d['value']/1e6,2), 'M nets/s', round(d['ms_per_step'],2), 'ms', round(d['roofline_step']['kernel_ms_per_step']['k_assign'],2))"
done; done
