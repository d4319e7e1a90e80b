# session 4: k_elmore via-stack change points; block kernel variants; parity under both Elmore kernels
set -x
mkdir -p gpurun_out
K="config_parity or config3_parity_full or config4_parity_sample or bitwise_fp or degenerate or layer_counts or ties or weight_regimes or sharded or nccl or full_size_oracle_hashes"
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "$K" 2>&1 | tail -3 > gpurun_out/s4f_pytest_blk.log
GAPLA_ELMORE_V2=1 timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "$K" 2>&1 | tail -3 > gpurun_out/s4f_pytest_v2.log
GAPLA_SO=libgapla_eb64.so GAPLA_EB_NODES=256 GAPLA_EB_SINKS=192 timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "config_parity or degenerate or ties or sharded" 2>&1 | tail -3 > gpurun_out/s4f_pytest_eb64.log
tail -n 3 gpurun_out/s4f_pytest_*.log
ab() {  # label env...
  L=$1; shift
  env "$@" timeout 600 python bench.py --config ${CFG:-5} --steps 10 --no-e2e --no-cpu-baseline --no-pre > gpurun_out/s4f_ab_$L.json 2> gpurun_out/s4f_ab_$L.err
  python -c "import json;d=json.load(open('gpurun_out/s4f_ab_$L.json'));k=d['roofline_step']['kernel_ms_per_step'];print('$L', d['ms_per_step'], 'elmore', k['k_elmore'])" || tail -2 gpurun_out/s4f_ab_$L.err
}
ab v2 GAPLA_ELMORE_V2=1
ab blk X=1
ab blk512 GAPLA_EB_NODES=512 GAPLA_EB_SINKS=384
ab eb64_384 GAPLA_SO=libgapla_eb64.so GAPLA_EB_NODES=384 GAPLA_EB_SINKS=320
ab eb64_256 GAPLA_SO=libgapla_eb64.so GAPLA_EB_NODES=256 GAPLA_EB_SINKS=192
ab eb64_192 GAPLA_SO=libgapla_eb64.so GAPLA_EB_NODES=192 GAPLA_EB_SINKS=160
CFG=4 ab v2_c4 GAPLA_ELMORE_V2=1
CFG=4 ab eb64_256_c4 GAPLA_SO=libgapla_eb64.so GAPLA_EB_NODES=256 GAPLA_EB_SINKS=192
GAPLA_ELMORE_V2=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_elmore -c 1 \
    -o gpurun_out/s4f_prof_v2 python bench.py --config 5 --ncu-pass --warmup 1 > gpurun_out/s4f_ncu1.log 2>&1
GAPLA_SO=libgapla_eb64.so GAPLA_EB_NODES=256 GAPLA_EB_SINKS=192 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_elmore_blk -c 1 \
    -o gpurun_out/s4f_prof_eb64 python bench.py --config 5 --ncu-pass --warmup 1 > gpurun_out/s4f_ncu2.log 2>&1
tail -n 1 gpurun_out/s4f_ncu1.log gpurun_out/s4f_ncu2.log
