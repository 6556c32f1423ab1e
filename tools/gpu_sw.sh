timeout 600 python tools/bench_conv.py --quick 2>&1 | tail -28 | cut -c1-160
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 1500 python tools/bench_configs.py --only c4 --no-cpu 2>&1 | tail -1
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-unfused 2>&1 | tail -1 | cut -c1-250
