# Round-2 evidence refresh (current HEAD): full GPU suite, smoke, default bench (cfg5 + e2e + CPU baselines),
# configs 1-4, paper batches, ncu launch list of one cfg5 step (+ pre-timing), compute-sanitizer of the new kernels
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1800 python -m pytest tests -q -m gpu --timeout 600 2>&1 | tail -5 > gpurun_out/f_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/f_cfg5_bench.json 2> gpurun_out/f_cfg5_bench.err
for C in 1 2 3 4; do
  timeout 900 python bench.py --config $C --no-cpu-baseline > gpurun_out/f_cfg${C}_bench.json 2> gpurun_out/f_cfg${C}_bench.err
done
timeout 900 python bench.py --batching paper --no-e2e --no-cpu-baseline --no-pre > gpurun_out/f_cfg5_bench_paper_batches.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --profile-from-start off --csv --log-file gpurun_out/f_cfg5_launches.csv python bench.py --ncu-pass --ncu-pre --warmup 1 \
    > gpurun_out/f_ncu_pass.log 2>&1
CS="compute-sanitizer --target-processes all --print-limit 50 --error-exitcode 9"
timeout 900 $CS --tool memcheck --leak-check no python tools/sanitize_run.py next2 bignets cfg1_batch > gpurun_out/f_sanitize_memcheck.log 2>&1
echo "memcheck rc=$?" > gpurun_out/f_sanitize_summary.txt
timeout 900 $CS --tool racecheck --racecheck-report all python tools/sanitize_run.py next2 > gpurun_out/f_sanitize_racecheck.log 2>&1
echo "racecheck rc=$?" >> gpurun_out/f_sanitize_summary.txt
timeout 900 $CS --tool synccheck python tools/sanitize_run.py next2 > gpurun_out/f_sanitize_synccheck.log 2>&1
echo "synccheck rc=$?" >> gpurun_out/f_sanitize_summary.txt
cat gpurun_out/f_pytest_gpu.log gpurun_out/f_smoke.log gpurun_out/f_sanitize_summary.txt
for C in 1 2 3 4 5; do python -c "import json;d=json.load(open('gpurun_out/f_cfg${C}_bench.json'));print($C, d['value']/1e6, d['ms_per_step'], d['e2e'] and d['e2e']['value'])"; done
