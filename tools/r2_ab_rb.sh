BNFF_F32_RB64=1 timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "f32" 2>&1 | tail -1
for v in 0 1 0 1; do
  BNFF_F32_RB64=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-unfused --also "" > gpurun_out/ab_rb$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_rb$v.json')); print('RB64=$v', round(d['ms_per_step'],3), d['step_profile']['kernel_shares'].get('fprop'))"
done
