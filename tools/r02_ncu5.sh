# ncu --set full of one mid-run cfg5 k_assign launch, group path vs warp path
for G in 1 0; do
GAPLA_GROUP=$G timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_assign -s 40 -c 1 \
    -o gpurun_out/prof5_g$G python bench.py --config 5 --ncu-pass --warmup 1 > gpurun_out/ncu5_g$G.log 2>&1
tail -n 2 gpurun_out/ncu5_g$G.log
done
