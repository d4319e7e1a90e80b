timeout 900 python tools/ablation.py --config 3 > gpurun_out/ablation_cfg3.jsonl 2> gpurun_out/ablation.err
cat gpurun_out/ablation_cfg3.jsonl; tail -3 gpurun_out/ablation.err
