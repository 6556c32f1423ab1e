timeout 1200 python -m pytest tests/test_dp_engine.py tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_dp.py -m gpu -q -x > gpurun_out/r2_quick.txt 2>&1
tail -2 gpurun_out/r2_quick.txt; grep -E "^(FAILED|E   )" gpurun_out/r2_quick.txt | head -10
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
tail -2 gpurun_out/r2_bench.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/r2_bench.json'))
print('f32', d['ms_per_step'], d['value'], d['e2e']['value'], d.get('speedup_vs_unfused'), d['roofline']['kernel'], d['roofline']['frac'])
b=d.get('bf16_mode', {})
print('bf16', b.get('ms_per_step'), b.get('value'), b.get('e2e',{}).get('value'), b.get('speedup_vs_unfused'))
print(d['step_profile']['kernel_shares']); print(b['step_profile']['kernel_shares'])
PY
timeout 600 python tools/profile_step.py --dtype f32 --level bnff+icf --top 10 > gpurun_out/prof_f32win.txt 2>&1; grep -A12 "by layer group" gpurun_out/prof_f32win.txt
