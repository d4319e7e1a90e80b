# Round-2 evidence refresh (current HEAD): full GPU suite, smoke, default bench (cfg5 + e2e + CPU baselines),
cat gpurun_out/f_pytest_gpu.log gpurun_out/f_smoke.log
for C in 1 2 3 4 5; do python -c "import json;d=json.load(open('gpurun_out/f_cfg${C}_bench.json'));print($C, d['value']/1e6, d['ms_per_step'], d['e2e'] and d['e2e']['value'])"; done
