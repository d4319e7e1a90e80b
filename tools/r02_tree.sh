# A/B of the pairwise (G', key) reduction in group_node (GROUP_TREE, libgapla_tr.so): parity of the variant, cfg5 / cfg3 / cfg4 timing
set -x
mkdir -p gpurun_out
GAPLA_SO=libgapla_tr.so timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "config_parity or config3_parity_full or hashes or layer_counts or random_state or weight_regimes or snapshot" 2>&1 | tail -4 > gpurun_out/t_pytest.log
cat gpurun_out/t_pytest.log
ab() {  # label config env...
  L=$1; C=$2; shift; shift
  env "$@" timeout 600 python bench.py --config $C --steps 10 --no-e2e --no-cpu-baseline --no-pre > gpurun_out/t_ab_${L}_$C.json 2> gpurun_out/t_ab_${L}_$C.err
  python -c "import json;d=json.load(open('gpurun_out/t_ab_${L}_$C.json'));k=d['roofline_step']['kernel_ms_per_step'];print('$L cfg$C', d['ms_per_step'], 'assign', k['k_assign'])"
}
for C in 5 3 4; do ab base $C X=1; ab tree $C GAPLA_SO=libgapla_tr.so; done
ab base 5 X=1
ab tree 5 GAPLA_SO=libgapla_tr.so
