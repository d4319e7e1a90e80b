# HEAD sanity on one B200: GPU parity suite, smoke, default bench (cfg5 with e2e + cpu baseline), cfg3/cfg4 quick
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu --timeout 400 2>&1 | tail -8 > gpurun_out/h_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h_smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/h_cfg5_bench.json 2> gpurun_out/h_cfg5_bench.err
for C in 3 4; do
  timeout 900 python bench.py --config $C --no-cpu-baseline > gpurun_out/h_cfg${C}_bench.json 2> gpurun_out/h_cfg${C}_bench.err
done
cat gpurun_out/h_pytest_gpu.log gpurun_out/h_smoke.log
for C in 3 4 5; do python -c "import json;d=json.load(open('gpurun_out/h_cfg${C}_bench.json'));print($C, d['value']/1e6, d['ms_per_step'], d['e2e'] and d['e2e']['value'])"; done
