for dt in f32 bf16; do
  timeout 900 ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r2_step_launches_$dt.csv python tools/ncu_step_bytes.py --dtype $dt --level bnff+icf > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/r2_step_launches_$dt.csv > gpurun_out/r2_step_launches_$dt.txt 2>&1
  head -25 gpurun_out/r2_step_launches_$dt.txt
done
timeout 1200 python -m pytest tests/test_gpu_models.py tests/test_gpu_parity.py -m gpu -q -k "resnet or c1 or tiny" > gpurun_out/r2_wide.txt 2>&1; tail -2 gpurun_out/r2_wide.txt
timeout 900 python tools/bench_configs.py --dtype bf16 --no-cpu --only c4 > gpurun_out/r2_c4_bf16.jsonl 2>&1; cut -c1-300 gpurun_out/r2_c4_bf16.jsonl
timeout 900 python tools/bench_configs.py --dtype f32 --no-cpu --only c4 > gpurun_out/r2_c4_f32.jsonl 2>&1; cut -c1-300 gpurun_out/r2_c4_f32.jsonl
timeout 1200 python tools/c5_sweep.py --time --out gpurun_out/r2_c5_time.json > gpurun_out/r2_c5.txt 2>&1; tail -30 gpurun_out/r2_c5.txt
