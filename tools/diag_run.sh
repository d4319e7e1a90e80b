for C in 1 2 4; do
  timeout 900 python bench.py --config $C --no-cpu-baseline > gpurun_out/bench_cfg$C.json 2> gpurun_out/bench_cfg$C.err
  python -c "import json;d=json.load(open('gpurun_out/bench_cfg$C.json'));print($C, d['value']/1e6, 'Mnets/s', d['ms_per_step'], 'ms', d['config']['batches'], 'batches', 'e2e', d['e2e']['value']/1e6)"
done
timeout 900 python bench.py --batching paper --no-e2e --no-cpu-baseline > gpurun_out/bench_paper_cfg5.json 2> gpurun_out/bench_paper_cfg5.err
python -c "import json;d=json.load(open('gpurun_out/bench_paper_cfg5.json'));print('paper', d['value']/1e6, d['ms_per_step'], d['config']['batches'], d['roofline_step']['kernel_ms_per_step'])"
