timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_window_strict.py -m gpu -q -x > gpurun_out/r2_fold.txt 2>&1
tail -2 gpurun_out/r2_fold.txt; grep -E "^(FAILED|E   )" gpurun_out/r2_fold.txt | head -10
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
tail -2 gpurun_out/r2_bench.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/r2_bench.json'))
print('f32', d['ms_per_step'], d['value'], d['e2e']['value'], d.get('speedup_vs_unfused'), d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['traffic'])
b=d.get('bf16_mode', {})
print('bf16', b.get('ms_per_step'), b.get('value'), b.get('e2e',{}).get('value'), b.get('speedup_vs_unfused'))
print(d['step_profile']['kernel_shares'])
PY
timeout 600 python tools/kernel_bw.py --json gpurun_out/kernel_bw.json > gpurun_out/kernel_bw.txt 2>&1; cat gpurun_out/kernel_bw.txt
