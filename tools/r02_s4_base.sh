# session-4 baseline at HEAD: e2e phase times (cfg5) and a short cfg5 bench
mkdir -p gpurun_out
GAPLA_VERBOSE=1 timeout 600 python tools/e2e_diag.py --config 5 > gpurun_out/s4_e2e_phases.log 2>&1
tail -30 gpurun_out/s4_e2e_phases.log
timeout 600 python bench.py --config 5 --steps 10 --no-cpu-baseline > gpurun_out/s4_base_cfg5.json 2> gpurun_out/s4_base_cfg5.err
python -c "import json;d=json.load(open('gpurun_out/s4_base_cfg5.json'));print(d['value']/1e6, d['ms_per_step'], d['roofline_step']['kernel_ms_per_step'], d['e2e'])"
