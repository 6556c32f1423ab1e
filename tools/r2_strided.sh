# stride-2 patch-matrix path: kernel + engine parity, ResNet-50 model parity, C4 A/B, step profile
timeout 300 python tools/strided_probe.py 2>&1 | grep -v Warn | tail -4
timeout 900 python -m pytest tests/test_gpu_strided.py -q -p no:randomly > gpurun_out/r2s_tests.txt 2>&1
tail -3 gpurun_out/r2s_tests.txt; grep "^FAILED" gpurun_out/r2s_tests.txt | head
timeout 900 python -m pytest tests/test_gpu_models.py tests/test_gpu_window_strict.py tests/test_gpu_parity.py -q -p no:randomly > gpurun_out/r2s_models.txt 2>&1
tail -3 gpurun_out/r2s_models.txt; grep "^FAILED" gpurun_out/r2s_models.txt | head
for dt in bf16 f32; do
  for on in 1; do
    BNFF_COL_STRIDED=$on timeout 600 python tools/bench_configs.py --only c4 --dtype $dt --no-cpu > gpurun_out/r2s_c4_${dt}_$on.jsonl 2>> gpurun_out/r2s_c4.err
    echo "$dt col=$on"; cat gpurun_out/r2s_c4_${dt}_$on.jsonl
  done
done
timeout 600 python tools/profile_step.py --model resnet50 --batch 128 --dtype bf16 --top 30 > gpurun_out/r2s_prof_bf16.txt 2>&1
head -60 gpurun_out/r2s_prof_bf16.txt
