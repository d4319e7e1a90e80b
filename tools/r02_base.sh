set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
cat gpurun_out/bench_cfg5.json
for C in 3 4; do
  timeout 900 python bench.py --config $C --no-e2e --no-cpu-baseline > gpurun_out/bench_q_cfg$C.json 2> gpurun_out/bench_q_cfg$C.err
  cat gpurun_out/bench_q_cfg$C.json
done
