timeout 600 python tools/bench_conv.py 2>&1 | grep -E "n64  56|worst" | cut -c1-150
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for i in 1 2 3; do timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu --no-unfused 2>&1 | tail -1 | cut -c170-240; done
