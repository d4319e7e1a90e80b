# session 4: k_elmore_blk (CTA-staged blocks, column layout) — GPU suite, A/B vs the thread-per-net k_elmore, ncu
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x ${PYK:-} 2>&1 | tail -6 > gpurun_out/s4e_pytest.log
cat gpurun_out/s4e_pytest.log
ab() {  # label env...
  L=$1; shift
  env "$@" timeout 600 python bench.py --config ${CFG:-5} --steps 10 --no-e2e --no-cpu-baseline --no-pre > gpurun_out/s4e_ab_$L.json 2> gpurun_out/s4e_ab_$L.err
  python -c "import json;d=json.load(open('gpurun_out/s4e_ab_$L.json'));k=d['roofline_step']['kernel_ms_per_step'];print('$L', d['ms_per_step'], 'elmore', k['k_elmore'])" || tail -2 gpurun_out/s4e_ab_$L.err
}
ab blk X=1
ab v2 GAPLA_ELMORE_V2=1
ab blk1024 GAPLA_EB_NODES=1024 GAPLA_EB_SINKS=768
ab blk512 GAPLA_EB_NODES=512 GAPLA_EB_SINKS=384
ab blk640 GAPLA_EB_NODES=640 GAPLA_EB_SINKS=512
CFG=4 ab blk_c4 X=1
CFG=4 ab v2_c4 GAPLA_ELMORE_V2=1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_elmore --csv \
    --log-file gpurun_out/s4e_elm_launches.csv python bench.py --config 5 --ncu-pass --warmup 1 > gpurun_out/s4e_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_elmore_blk -c 1 \
    -o gpurun_out/s4e_prof_elmblk python bench.py --config 5 --ncu-pass --warmup 1 > gpurun_out/s4e_ncu2.log 2>&1
tail -n 2 gpurun_out/s4e_ncu1.log gpurun_out/s4e_ncu2.log
