# session 4: e2e phases after the host builder changes (neighbour arrays, reserved chunk arrays); GPU suite; cfg5 bench with e2e
mkdir -p gpurun_out
GAPLA_VERBOSE=1 timeout 600 python tools/e2e_diag.py --config 5 > gpurun_out/s4j_e2e_phases.log 2>&1
grep -E "rep|build threads" gpurun_out/s4j_e2e_phases.log
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -4 > gpurun_out/s4j_pytest.log
cat gpurun_out/s4j_pytest.log
timeout 900 python bench.py --config 5 --steps 10 --no-cpu-baseline > gpurun_out/s4j_cfg5.json 2> gpurun_out/s4j_cfg5.err
python -c "import json;d=json.load(open('gpurun_out/s4j_cfg5.json'));print(d['value']/1e6, d['ms_per_step'], d['roofline_step']['kernel_ms_per_step'], d['e2e']['seconds_per_step'], d['e2e']['value']/1e6)"
