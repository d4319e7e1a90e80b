# NEXT #2 on the GPU: parity of k_pre_timing / GPU Alg. 1, then cfg3 + cfg5 quick benches with the pre_assignment block
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_pre_timing.py -q -m gpu -x 2>&1 | tail -15 > gpurun_out/n2_pytest.log
cat gpurun_out/n2_pytest.log
for C in 3 5; do
  timeout 900 python bench.py --config $C --no-e2e --no-cpu-baseline > gpurun_out/n2_cfg$C.json 2> gpurun_out/n2_cfg$C.err
  python -c "import json;d=json.load(open('gpurun_out/n2_cfg$C.json'));print($C, d['value']/1e6, d['ms_per_step'], json.dumps(d['pre_assignment']))"
  tail -3 gpurun_out/n2_cfg$C.err
done
