# session 4: k_elmore CTA size (ELM_T 128 / 64 / 32, and 64 with an 80-register bound) A/B at configs 5 and 4; parity of the variants
mkdir -p gpurun_out
ab() {  # label env...
  L=$1; shift
  env "$@" timeout 600 python bench.py --config ${CFG:-5} --steps 10 --no-e2e --no-cpu-baseline --no-pre > gpurun_out/s4k_ab_$L.json 2> gpurun_out/s4k_ab_$L.err
  python -c "import json;d=json.load(open('gpurun_out/s4k_ab_$L.json'));k=d['roofline_step']['kernel_ms_per_step'];print('$L', d['ms_per_step'], 'elmore', k['k_elmore'])" || tail -2 gpurun_out/s4k_ab_$L.err
}
ab t128 X=1
ab t64 GAPLA_SO=libgapla_et64.so
ab t32 GAPLA_SO=libgapla_et32.so
ab t64m GAPLA_SO=libgapla_et64m.so
ab t128b X=1
CFG=4 ab t128_c4 X=1
CFG=4 ab t64_c4 GAPLA_SO=libgapla_et64.so
CFG=4 ab t64m_c4 GAPLA_SO=libgapla_et64m.so
for V in et64 et64m; do
  GAPLA_SO=libgapla_$V.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "config_parity or degenerate or ties or sharded or full_size_oracle_hashes" 2>&1 | tail -1
done
