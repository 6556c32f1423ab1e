mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 900 python tools/traffic_ledger.py > gpurun_out/traffic_ledger.txt 2>&1; cat gpurun_out/traffic_ledger.txt
timeout 1200 python -m paper_1807_01702_b200.cli bench --model densenet-121 --batch 64 --fusion all --iters 10 --warmup 3 --out gpurun_out/bench_d121_levels.csv 2>&1 | tail -7
