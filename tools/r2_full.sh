rm -f gpurun_out/parity_models.jsonl
BNFF_PARITY_LOG=$PWD/gpurun_out/parity_models.jsonl timeout 2400 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/r2_full.txt 2>&1
grep -E "passed|failed" gpurun_out/r2_full.txt | tail -2; grep -E "^FAILED" gpurun_out/r2_full.txt | head -30
timeout 1200 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
tail -2 gpurun_out/r2_bench.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/r2_bench.json'))
print('f32', d['ms_per_step'], d['value'], d['e2e']['value'], d.get('speedup_vs_unfused'), d['roofline']['kernel'], d['roofline']['frac'])
b=d.get('bf16_mode', {})
print('bf16', b.get('ms_per_step'), b.get('value'), b.get('e2e',{}).get('value'), b.get('speedup_vs_unfused'), b.get('roofline',{}).get('kernel'), b.get('roofline',{}).get('frac'))
print('cpu', d.get('cpu_baseline'))
PY
