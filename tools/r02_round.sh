# Round-2 evidence on one B200 (all outputs under gpurun_out/r02_*): GPU parity suite, smoke, the
# default bench (cfg5: e2e + cpu_baseline), configs 1-4, Alg. 1 snapshot batches, the ncu launch
# list of one cfg5 step (+dram bytes), ncu --set full of a mid-step k_assign_g launch, k_elmore and
# k_eval_plane, and compute-sanitizer over tools/sanitize_run.py.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -q -m gpu --timeout 300 2>&1 | tail -5 > gpurun_out/r02_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/r02_cfg5_bench.json 2> gpurun_out/r02_cfg5_bench.err
for C in 1 2 3 4; do
  timeout 900 python bench.py --config $C --no-cpu-baseline > gpurun_out/r02_cfg${C}_bench.json 2> gpurun_out/r02_cfg${C}_bench.err
done
timeout 900 python bench.py --batching paper --no-e2e --no-cpu-baseline > gpurun_out/r02_cfg5_bench_paper_batches.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --profile-from-start off --csv --log-file gpurun_out/r02_cfg5_launches.csv python bench.py --ncu-pass --warmup 1 \
    > gpurun_out/r02_ncu_pass.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_assign -s 40 -c 1 \
    -o gpurun_out/r02_prof_assign_cfg5 python bench.py --ncu-pass --warmup 1 > gpurun_out/r02_ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_elmore -c 1 \
    -o gpurun_out/r02_prof_elmore_cfg5 python bench.py --ncu-pass --warmup 1 >> gpurun_out/r02_ncu_full.log 2>&1
CS="compute-sanitizer --target-processes all --print-limit 50 --error-exitcode 9"
timeout 1500 $CS --tool memcheck --leak-check no python tools/sanitize_run.py > gpurun_out/r02_sanitize_memcheck.log 2>&1
echo "memcheck rc=$?" > gpurun_out/r02_sanitize_summary.txt
timeout 1500 $CS --tool synccheck python tools/sanitize_run.py cfg1_batch cfg1_flow bignets snapshot group_paths nccl_one_gpu > gpurun_out/r02_sanitize_synccheck.log 2>&1
echo "synccheck rc=$?" >> gpurun_out/r02_sanitize_summary.txt
timeout 2400 $CS --tool racecheck --racecheck-report all python tools/sanitize_run.py cfg1_batch bignets snapshot group_paths > gpurun_out/r02_sanitize_racecheck.log 2>&1
echo "racecheck rc=$?" >> gpurun_out/r02_sanitize_summary.txt
cat gpurun_out/r02_pytest_gpu.log gpurun_out/r02_smoke.log gpurun_out/r02_sanitize_summary.txt
for C in 1 2 3 4 5; do python -c "import json;d=json.load(open('gpurun_out/r02_cfg${C}_bench.json'));print($C, d['value']/1e6, d['ms_per_step'], d['e2e'] and d['e2e']['value'])"; done
