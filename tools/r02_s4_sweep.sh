# session 4: batch-tail knobs (team/group split per batch) on configs 3 / 4 / 5
mkdir -p gpurun_out
ab() {  # label cfg env...
  L=$1; C=$2; shift; shift
  env "$@" timeout 600 python bench.py --config $C --steps 10 --no-e2e --no-cpu-baseline --no-pre > gpurun_out/s4s_$L.json 2> gpurun_out/s4s_$L.err
  python -c "import json;d=json.load(open('gpurun_out/s4s_$L.json'));print('$L', d['ms_per_step'])" || tail -2 gpurun_out/s4s_$L.err
}
for C in 3 4; do
  ab base_c$C $C X=1
  ab lat4_c$C $C GAPLA_GROUP_NMAX_LAT=4
  ab lat6_c$C $C GAPLA_GROUP_NMAX_LAT=6
  ab lat12_c$C $C GAPLA_GROUP_NMAX_LAT=12
  ab ppw4_c$C $C GAPLA_NMAX_NETS_PER_WARP=4
  ab ppw16_c$C $C GAPLA_NMAX_NETS_PER_WARP=16
  ab split1_c$C $C GAPLA_BIG_SPLIT=1
  ab split0_c$C $C GAPLA_BIG_SPLIT=0
done
ab base_c5 5 X=1
ab lat6_c5 5 GAPLA_GROUP_NMAX_LAT=6
ab ppw16_c5 5 GAPLA_NMAX_NETS_PER_WARP=16
