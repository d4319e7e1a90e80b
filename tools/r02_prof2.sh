timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_assign -s ${SKIP:-40} -c 1 \
    -o gpurun_out/prof5 python bench.py --config 5 --ncu-pass --warmup 1 > gpurun_out/ncu5.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_assign -s 60 -c 1 \
    -o gpurun_out/prof4 python bench.py --config 4 --ncu-pass --warmup 1 > gpurun_out/ncu4.log 2>&1
tail -n 1 gpurun_out/ncu5.log gpurun_out/ncu4.log
