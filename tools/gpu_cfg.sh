mkdir -p gpurun_out
timeout 1500 python tools/bench_configs.py --only c4 > gpurun_out/configs_c4.jsonl 2> gpurun_out/configs.err; cat gpurun_out/configs_c4.jsonl; tail -5 gpurun_out/configs.err
