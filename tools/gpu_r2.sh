mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python tools/ablate.py --level bnff+icf > gpurun_out/ablate_icf.txt 2>&1; cat gpurun_out/ablate_icf.txt
timeout 600 python bench.py --steps 10 --warmup 3 --level bnff+icf --no-cpu --no-unfused > gpurun_out/bench_icf.log 2>&1; tail -1 gpurun_out/bench_icf.log | cut -c1-300
timeout 600 python tools/profile_step.py --level bnff+icf --top 30 > gpurun_out/prof_icf.txt 2>&1; head -50 gpurun_out/prof_icf.txt
