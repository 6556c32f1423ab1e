mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log; grep -E "^E  |FAIL" gpurun_out/pytest_gpu.log | head -20
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-unfused > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-300
timeout 600 python tools/profile_step.py --top 5 > gpurun_out/prof_icf.txt 2>&1; head -50 gpurun_out/prof_icf.txt
