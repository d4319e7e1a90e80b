# parity suite, then A/B of k_assign_g (group path) vs k_assign (GAPLA_GROUP=0) on cfg3 with ncu source capture
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
tail -25 gpurun_out/pytest_gpu.log
CFG=${CFG:-3}
for G in 1 0; do
  GAPLA_GROUP=$G timeout 900 python bench.py --config $CFG --no-e2e --no-cpu-baseline > gpurun_out/bench_g${G}_cfg$CFG.json 2> gpurun_out/bench_g${G}_cfg$CFG.err
  python -c "import json;d=json.load(open('gpurun_out/bench_g${G}_cfg$CFG.json'));print('group=$G', d['value']/1e6, 'M nets/s', d['ms_per_step'], 'ms', d['roofline_step']['kernel_ms_per_step'])"
done
GAPLA_GROUP=1 timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_assign -s 40 -c 1 \
    -o gpurun_out/prof_g1_cfg$CFG python bench.py --config $CFG --ncu-pass --warmup 1 > gpurun_out/ncu_g1.log 2>&1
GAPLA_GROUP=0 timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_assign -s 40 -c 1 \
    -o gpurun_out/prof_g0_cfg$CFG python bench.py --config $CFG --ncu-pass --warmup 1 > gpurun_out/ncu_g0.log 2>&1
tail -3 gpurun_out/ncu_g1.log gpurun_out/ncu_g0.log
