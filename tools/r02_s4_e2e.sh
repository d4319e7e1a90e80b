# session 4: e2e phase times (cfg5) after the host-side changes (GPU la_get_solution, background forest upload); GPU suite
mkdir -p gpurun_out
GAPLA_VERBOSE=1 timeout 600 python tools/e2e_diag.py --config 5 > gpurun_out/s4i_e2e_phases.log 2>&1
grep -E "rep|solution\]" gpurun_out/s4i_e2e_phases.log
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -4 > gpurun_out/s4i_pytest.log
cat gpurun_out/s4i_pytest.log
