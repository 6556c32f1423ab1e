# GPU validation + bench pass (used via gpurun): tests, smoke, bench, step profile
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-700
timeout 600 python tools/profile_step.py --top 40 > gpurun_out/prof_bnff.txt 2>&1; head -45 gpurun_out/prof_bnff.txt
