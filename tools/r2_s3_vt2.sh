mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_models.py -m gpu -q -p no:randomly -x > gpurun_out/s3vt2_tests.txt 2>&1
tail -2 gpurun_out/s3vt2_tests.txt; grep -E "^FAILED" gpurun_out/s3vt2_tests.txt | head
bash tools/gpu_abn.sh B D > gpurun_out/s3vt2_ab.txt 2>&1; cat gpurun_out/s3vt2_ab.txt
timeout 900 ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/s3vt2_launches_f32.csv python tools/ncu_step_bytes.py --dtype f32 --level bnff+icf > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/s3vt2_launches_f32.csv > gpurun_out/s3vt2_launches_f32.txt 2>&1; head -12 gpurun_out/s3vt2_launches_f32.txt
bash tools/r2_s3_ncu33.sh
