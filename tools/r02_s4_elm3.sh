# session 4: k_elmore with next-node prefetch and dynamic T columns; register-bound variants
set -x
mkdir -p gpurun_out
K="config_parity or config4_parity_sample or bitwise_fp or degenerate or ties or sharded or nccl or full_size_oracle_hashes"
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "$K" 2>&1 | tail -3 > gpurun_out/s4g_pytest.log
GAPLA_SO=libgapla_em6.so timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "config_parity or degenerate or ties" 2>&1 | tail -3 > gpurun_out/s4g_pytest_em6.log
tail -n 3 gpurun_out/s4g_pytest*.log
ab() {  # label env...
  L=$1; shift
  env "$@" timeout 600 python bench.py --config ${CFG:-5} --steps 10 --no-e2e --no-cpu-baseline --no-pre > gpurun_out/s4g_ab_$L.json 2> gpurun_out/s4g_ab_$L.err
  python -c "import json;d=json.load(open('gpurun_out/s4g_ab_$L.json'));k=d['roofline_step']['kernel_ms_per_step'];print('$L', d['ms_per_step'], 'elmore', k['k_elmore'])" || tail -2 gpurun_out/s4g_ab_$L.err
}
ab pf X=1
ab em6 GAPLA_SO=libgapla_em6.so
ab em8 GAPLA_SO=libgapla_em8.so
ab pf2 X=1
CFG=4 ab pf_c4 X=1
CFG=4 ab em6_c4 GAPLA_SO=libgapla_em6.so
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_elmore -c 1 \
    -o gpurun_out/s4g_prof_pf python bench.py --config 5 --ncu-pass --warmup 1 > gpurun_out/s4g_ncu1.log 2>&1
tail -n 1 gpurun_out/s4g_ncu1.log
