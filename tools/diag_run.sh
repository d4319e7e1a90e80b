timeout 1200 python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
timeout 900 python bench.py --config 3 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
python -c "
import json
for c in ('cfg5','cfg3'):
    d=json.load(open(f'gpurun_out/bench_{c}.json'))
    print(c, round(d['value']/1e6,2), round(d['ms_per_step'],1), 'e2e', round(d['e2e']['value']/1e6,3), 'launches', d['gpu_launches'], d['clocks'])
"
