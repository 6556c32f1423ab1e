timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_pins.py -m gpu -q -x -k "f32 or fused_equals" 2>&1 | tail -1
for v in 32 16 32 16; do
  BNFF_WG32_KB=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-unfused --also "" > gpurun_out/ab_kb$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_kb$v.json')); print('KB=$v', round(d['ms_per_step'],3), d['step_profile']['kernel_shares'].get('wgrad'))"
done
