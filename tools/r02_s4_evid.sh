# Round-2 session-4 evidence at HEAD on one B200 (outputs gpurun_out/s4z_*): GPU suite (gate), smoke,
# default bench (cfg5: e2e + cpu baselines), configs 1-4, Alg. 1 snapshot batches, e2e phases, the ncu
# launch list of one cfg5 step (+ DRAM bytes), ncu --set full of a mid-step k_assign_g launch and k_elmore.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -q -m gpu --timeout 300 2>&1 | tail -5 > gpurun_out/s4z_pytest_gpu.log
cat gpurun_out/s4z_pytest_gpu.log
grep -q " passed" gpurun_out/s4z_pytest_gpu.log && ! grep -q "failed\|error" gpurun_out/s4z_pytest_gpu.log || { echo "GPU suite not green: stop"; exit 3; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4z_smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/s4z_cfg5_bench.json 2> gpurun_out/s4z_cfg5_bench.err
for C in 1 2 3 4; do
  timeout 900 python bench.py --config $C --no-cpu-baseline > gpurun_out/s4z_cfg${C}_bench.json 2> gpurun_out/s4z_cfg${C}_bench.err
done
timeout 900 python bench.py --batching paper --no-e2e --no-cpu-baseline > gpurun_out/s4z_cfg5_bench_paper_batches.json 2>/dev/null
GAPLA_VERBOSE=1 timeout 600 python tools/e2e_diag.py --config 5 > gpurun_out/s4z_e2e_phases.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --profile-from-start off --csv --log-file gpurun_out/s4z_cfg5_launches.csv python bench.py --ncu-pass --warmup 1 \
    > gpurun_out/s4z_ncu_pass.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_assign -s 40 -c 1 \
    -o gpurun_out/s4z_prof_assign_cfg5 python bench.py --ncu-pass --warmup 1 > gpurun_out/s4z_ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_elmore -c 1 \
    -o gpurun_out/s4z_prof_elmore_cfg5 python bench.py --ncu-pass --warmup 1 >> gpurun_out/s4z_ncu_full.log 2>&1
cat gpurun_out/s4z_smoke.log
for C in 1 2 3 4 5; do python -c "import json;d=json.load(open('gpurun_out/s4z_cfg${C}_bench.json'));print($C, d['value']/1e6, d['ms_per_step'], d['e2e'] and d['e2e']['value'])"; done
grep -E "^rep" gpurun_out/s4z_e2e_phases.log
