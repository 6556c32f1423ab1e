timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_window_strict.py -m gpu -q -x 2>&1 | tail -1
for dt in f32 bf16; do for v in 1 4 8 1 4 8; do
  BNFF_WG_MINKPT=$v timeout 600 python bench.py --dtype $dt --steps 20 --warmup 5 --no-cpu --no-unfused --also "" > gpurun_out/ab_kpt.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_kpt.json')); print('$dt minkpt=$v', round(d['ms_per_step'],3), d['step_profile']['kernel_shares'].get('wgrad'))"
done; done
