# parity suite (per-test timeout), then A/B of k_assign_g (group path) vs k_assign (GAPLA_GROUP=0)
set -x
mkdir -p gpurun_out
timeout ${TTIME:-1500} python -m pytest ${TESTS:-tests} -x -q -m gpu --timeout 300 ${PYARGS:-} 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
tail -30 gpurun_out/pytest_gpu.log
for CFG in ${CFGS:-3 5}; do
for G in ${GROUPS_AB:-1 0}; do
  GAPLA_GROUP=$G timeout 900 python bench.py --config $CFG --no-e2e --no-cpu-baseline > gpurun_out/bench_g${G}_cfg$CFG.json 2> gpurun_out/bench_g${G}_cfg$CFG.err
  python -c "import json;d=json.load(open('gpurun_out/bench_g${G}_cfg$CFG.json'));print('cfg$CFG group=$G', d['value']/1e6, 'M nets/s', d['ms_per_step'], 'ms', d['roofline_step']['kernel_ms_per_step'])" || tail -5 gpurun_out/bench_g${G}_cfg$CFG.err
done
done
if [ -n "$NCU" ]; then
GAPLA_GROUP=1 timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_assign -s 40 -c 1 \
    -o gpurun_out/prof_g1_cfg3 python bench.py --config 3 --ncu-pass --warmup 1 > gpurun_out/ncu_g1.log 2>&1
tail -n 3 gpurun_out/ncu_g1.log
fi
