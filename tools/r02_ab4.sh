for SO in libgapla_g44.so libgapla_g44b.so libgapla_g33.so libgapla_g22.so; do
for CFG in 3 5; do
  GAPLA_SO=$SO timeout 900 python bench.py --config $CFG --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/b.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b.json'));print('$SO cfg$CFG', round(d['value']/1e6,2), 'M nets/s', round(d['ms_per_step'],2), 'ms', round(d['roofline_step']['kernel_ms_per_step']['k_assign'],2))"
done; done
for NM in 8 16 24; do for CFG in 3 5; do
  GAPLA_GROUP_NMAX=$NM GAPLA_SO=libgapla_g44.so timeout 900 python bench.py --config $CFG --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/b.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b.json'));print('g44 nmax=$NM cfg$CFG', round(d['value']/1e6,2), 'M nets/s', round(d['ms_per_step'],2), 'ms', round(d['roofline_step']['kernel_ms_per_step']['k_assign'],2))"
done; done
