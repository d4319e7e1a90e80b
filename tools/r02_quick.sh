# parity suite + short benches (no e2e / cpu baseline); CFGS selects configs, TESTS the pytest selection
set -x
mkdir -p gpurun_out
timeout ${TTIME:-1200} python -m pytest ${TESTS:-tests} -x -q -m gpu ${PYARGS:-} 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
tail -25 gpurun_out/pytest_gpu.log
for C in ${CFGS:-3 5}; do
  timeout 900 python bench.py --config $C --no-e2e --no-cpu-baseline > gpurun_out/bench_q_cfg$C.json 2> gpurun_out/bench_q_cfg$C.err
  python -c "import json;d=json.load(open('gpurun_out/bench_q_cfg$C.json'));print($C, d['value']/1e6, 'M nets/s', d['ms_per_step'], 'ms', d['roofline_step']['kernel_ms_per_step'])"
  tail -3 gpurun_out/bench_q_cfg$C.err
done
