mkdir -p gpurun_out
timeout 600 python tools/bench_conv.py > gpurun_out/bench_conv.txt 2>&1; cat gpurun_out/bench_conv.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log; grep -E "^E  |FAIL" gpurun_out/pytest_gpu.log | head -20
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-400
timeout 600 python tools/profile_step.py --top 25 > gpurun_out/prof_icf.txt 2>&1; head -50 gpurun_out/prof_icf.txt
