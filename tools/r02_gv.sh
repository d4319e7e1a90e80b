# A/B of the vectorised per-node via-word gather (GATHER_VEC, libgapla_gv.so)
set -x
mkdir -p gpurun_out
GAPLA_SO=libgapla_gv.so timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "config_parity or config3_parity_full or hashes or layer_counts or random_state" 2>&1 | tail -4 > gpurun_out/g_pytest.log
cat gpurun_out/g_pytest.log
ab() {  # label config env...
  L=$1; C=$2; shift; shift
  env "$@" timeout 600 python bench.py --config $C --steps 10 --no-e2e --no-cpu-baseline --no-pre > gpurun_out/g_ab_${L}_$C.json 2> gpurun_out/g_ab_${L}_$C.err
  python -c "import json;d=json.load(open('gpurun_out/g_ab_${L}_$C.json'));k=d['roofline_step']['kernel_ms_per_step'];print('$L cfg$C', d['ms_per_step'], 'assign', k['k_assign'])"
}
for C in 5 3 4; do ab base $C X=1; ab gv $C GAPLA_SO=libgapla_gv.so; done
