mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log; grep -E "^E  |FAIL" gpurun_out/pytest_gpu.log | head -20
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-300
