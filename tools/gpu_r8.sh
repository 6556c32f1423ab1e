mkdir -p gpurun_out
timeout 600 python tools/bench_conv.py > gpurun_out/bench_conv.txt 2>&1; grep -E "56\^2|28\^2|14\^2|7\^2|worst" gpurun_out/bench_conv.txt | cut -c1-150
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log; grep -E "^E  |FAIL" gpurun_out/pytest_gpu.log | head -20
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-unfused > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-300
for c in 25 23; do echo "=== case $c"; timeout 120 python tools/trace_conv.py --only $c 2>&1 | tail -24 | head -12; done
