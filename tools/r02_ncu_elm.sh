timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_elmore -c 1 \
    -o gpurun_out/prof_elm5 python bench.py --config 5 --ncu-pass --warmup 1 > gpurun_out/ncu_elm.log 2>&1
tail -n 1 gpurun_out/ncu_elm.log
