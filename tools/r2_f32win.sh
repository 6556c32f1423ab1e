timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_pins.py -m gpu -q -x -k "f32 or fused_equals or cancellation or constant or tiny_full or stem or multistep" > gpurun_out/r2_f32win.txt 2>&1
tail -3 gpurun_out/r2_f32win.txt; grep -E "^(FAILED|E  )" gpurun_out/r2_f32win.txt | head -20
timeout 600 python bench.py --dtype f32 --also "" --steps 10 --warmup 3 --no-cpu > gpurun_out/r2_f32win_bench.json 2> gpurun_out/r2_f32win_bench.err
tail -2 gpurun_out/r2_f32win_bench.err; python -c "
import json; d=json.load(open('gpurun_out/r2_f32win_bench.json')); print(d['ms_per_step'], d['value'], d.get('speedup_vs_unfused'), d['step_profile']['kernel_shares'])"
timeout 600 python tools/profile_step.py --dtype f32 --level bnff+icf --top 30 > gpurun_out/prof_f32win.txt 2>&1; head -50 gpurun_out/prof_f32win.txt
