# Round-2 session-4 check of HEAD after the load-phase changes: GPU suite, smoke, default bench, config 3/4, e2e phases
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -q -m gpu --timeout 300 2>&1 | tail -5 > gpurun_out/s4r_pytest_gpu.log
cat gpurun_out/s4r_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4r_smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/s4r_cfg5_bench.json 2> gpurun_out/s4r_cfg5_bench.err
for C in 3 4; do timeout 900 python bench.py --config $C --no-cpu-baseline > gpurun_out/s4r_cfg${C}_bench.json 2> gpurun_out/s4r_cfg${C}_bench.err; done
GAPLA_VERBOSE=1 timeout 600 python tools/e2e_diag.py --config 5 > gpurun_out/s4r_e2e_phases.log 2>&1
cat gpurun_out/s4r_smoke.log
for C in 3 4 5; do python -c "import json;d=json.load(open('gpurun_out/s4r_cfg${C}_bench.json'));print($C, d['value']/1e6, d['ms_per_step'], d['e2e'] and d['e2e']['value'], d['e2e'] and d['e2e']['seconds_per_step'])"; done
grep -E "^rep|gapla load\]" gpurun_out/s4r_e2e_phases.log | tail -22
