timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_pins.py -m gpu -q -x -k "f32 or fused_equals" 2>&1 | tail -2
for v in 64 128 64 128; do
  BNFF_WG32_BN=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-unfused --also "" > gpurun_out/ab_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_$v.json')); print('BN=$v', round(d['ms_per_step'],3), d['roofline']['kernel'], round(d['step_profile']['kernel_shares'].get('wgrad',0),3))"
done
timeout 900 python -m pytest tests/test_gpu_models.py tests/test_gpu_parity.py -m gpu -q -k "resnet or c1 or tiny or multistep" 2>&1 | tail -2
timeout 1200 python tools/c5_sweep.py --time --out gpurun_out/r2_c5_time.json > gpurun_out/r2_c5.txt 2>&1; grep -E '"C": (512|1024)' gpurun_out/r2_c5.txt
