# thread-per-net k_elmore with shared-memory node values: parity subset, A/B (round-1 kernel, ELM_LOCAL 8/12/20), pre-timing v1 vs chunks
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_pre_timing.py -q -m gpu -x -k "not full_scale and not hash and not cfg3_sampled" 2>&1 | tail -4 > gpurun_out/e4_pytest.log
cat gpurun_out/e4_pytest.log
ab() {  # label env...
  L=$1; shift
  env "$@" timeout 600 python bench.py --config 5 --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/e4_ab_$L.json 2> gpurun_out/e4_ab_$L.err
  python -c "import json;d=json.load(open('gpurun_out/e4_ab_$L.json'));k=d['roofline_step']['kernel_ms_per_step'];print('$L', d['ms_per_step'], 'elmore', k['k_elmore'], 'pre', d['pre_assignment']['pre_timing']['ms'])"
}
ab v1 GAPLA_ELMORE_V1=1 GAPLA_PRE_V1=1
ab l12 X=1
ab l8 GAPLA_SO=libgapla_l8.so
ab l6 GAPLA_SO=libgapla_l6.so
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:'k_elmore|k_pre_timing' -c 2 \
    -o gpurun_out/e4_prof_cfg5 python bench.py --ncu-pass --ncu-pre --warmup 1 > gpurun_out/e4_ncu.log 2>&1
echo ncu rc=$?
