set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py --dtype f32 --steps 5 --warmup 3 --no-cpu > gpurun_out/r2p_f32.json 2> gpurun_out/r2p_f32.err
tail -3 gpurun_out/r2p_f32.err
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-unfused > gpurun_out/r2p_bf16.json 2> gpurun_out/r2p_bf16.err
tail -3 gpurun_out/r2p_bf16.err
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2p_pytest.txt 2>&1
tail -5 gpurun_out/r2p_pytest.txt
