# one ncu --set full capture of k_assign (and k_elmore) on the bench's ncu pass
CFG=${1:-3}
set -x
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_assign -c 1 \
    -o gpurun_out/prof_assign_cfg$CFG python bench.py --config $CFG --ncu-pass --warmup 1 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_elmore -c 1 \
    -o gpurun_out/prof_elmore_cfg$CFG python bench.py --config $CFG --ncu-pass --warmup 1 >> gpurun_out/ncu_full.log 2>&1
tail -5 gpurun_out/ncu_full.log
