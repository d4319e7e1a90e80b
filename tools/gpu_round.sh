# Round deliverables on one B200: GPU parity suite, smoke, the default bench (cfg5, with e2e and
# cpu_baseline), the cfg3 bench, the ncu launch list (+dram bytes) of one cfg5 step, and one
# ncu --set full capture of a mid-run k_assign launch and of k_elmore.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
timeout 600 python bench.py --config 3 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --profile-from-start off --csv --log-file gpurun_out/launches_cfg5.csv python bench.py --ncu-pass --warmup 1 \
    > gpurun_out/ncu_pass.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_assign -s 40 -c 1 \
    -o gpurun_out/prof_assign_cfg5 python bench.py --ncu-pass --warmup 1 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_elmore -c 1 \
    -o gpurun_out/prof_elmore_cfg5 python bench.py --ncu-pass --warmup 1 >> gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; cat gpurun_out/bench_cfg5.json gpurun_out/bench_cfg3.json
