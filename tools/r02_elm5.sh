# k_elmore with shared-memory node values: ELM_LOCAL 4 / 6 / 12, 6 CTAs/SM; pre-timing (windowed bigger nets); parity subset
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_pre_timing.py -q -m gpu -x -k "not full_scale and not hash and not cfg3_sampled" 2>&1 | tail -4 > gpurun_out/e5_pytest.log
cat gpurun_out/e5_pytest.log
ab() {  # label env...
  L=$1; shift
  env "$@" timeout 600 python bench.py --config 5 --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/e5_ab_$L.json 2> gpurun_out/e5_ab_$L.err
  python -c "import json;d=json.load(open('gpurun_out/e5_ab_$L.json'));k=d['roofline_step']['kernel_ms_per_step'];print('$L', d['ms_per_step'], 'elmore', k['k_elmore'], 'pre', d['pre_assignment']['pre_timing']['ms'])"
}
ab v1 GAPLA_ELMORE_V1=1
ab l12 X=1
ab l6 GAPLA_SO=libgapla_l6.so
ab l4 GAPLA_SO=libgapla_l4.so
ab l6m6 GAPLA_SO=libgapla_l6m6.so
