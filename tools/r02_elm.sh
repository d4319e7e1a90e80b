# chunked k_elmore: parity, A/B against the round-1 kernel and the two register budgets, ncu of the new kernels
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_pre_timing.py -q -m gpu -x 2>&1 | tail -8 > gpurun_out/e_pytest.log
cat gpurun_out/e_pytest.log
ab() {  # label env...
  L=$1; shift
  env "$@" timeout 600 python bench.py --config 5 --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/e_ab_$L.json 2> gpurun_out/e_ab_$L.err
  python -c "import json;d=json.load(open('gpurun_out/e_ab_$L.json'));k=d['roofline_step']['kernel_ms_per_step'];print('$L', d['ms_per_step'], 'elmore', k['k_elmore'], 'pre', d['pre_assignment']['pre_timing']['ms'])"
}
ab v1 GAPLA_ELMORE_V1=1
ab minb3 X=1
ab minb2 GAPLA_SO=libgapla_e2.so
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:'k_elmore|k_pre_timing' -c 2 \
    -o gpurun_out/e_prof_cfg5 python bench.py --ncu-pass --ncu-pre --warmup 1 > gpurun_out/e_ncu.log 2>&1
echo ncu rc=$?
