# A/B of the team dataflow (TEAM_FLOW, libgapla_tf.so): done-flags per node instead of a barrier per height level
set -x
mkdir -p gpurun_out
GAPLA_SO=libgapla_tf.so timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "config_parity or config3_parity_full or config4_parity or hashes or layer_counts or random_state or snapshot or variants or dense" 2>&1 | tail -4 > gpurun_out/tf_pytest.log
cat gpurun_out/tf_pytest.log
ab() {  # label config env...
  L=$1; C=$2; shift; shift
  env "$@" timeout 600 python bench.py --config $C --steps 10 --no-e2e --no-cpu-baseline --no-pre > gpurun_out/tf_ab_${L}_$C.json 2> gpurun_out/tf_ab_${L}_$C.err
  python -c "import json;d=json.load(open('gpurun_out/tf_ab_${L}_$C.json'));k=d['roofline_step']['kernel_ms_per_step'];print('$L cfg$C', d['ms_per_step'], 'assign', k['k_assign'])"
}
for C in 4 3 5; do ab base $C X=1; ab tf $C GAPLA_SO=libgapla_tf.so; done
