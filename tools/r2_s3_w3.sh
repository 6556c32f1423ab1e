mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/s3w3_tests.txt 2>&1
tail -2 gpurun_out/s3w3_tests.txt; grep -E "^FAILED" gpurun_out/s3w3_tests.txt | head
bash tools/gpu_env_ab2.sh BNFF_WRES3 f32 0 1 > gpurun_out/s3w3_ab.txt 2>&1; cat gpurun_out/s3w3_ab.txt
timeout 900 ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/s3w3_launches_f32.csv python tools/ncu_step_bytes.py --dtype f32 --level bnff+icf > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/s3w3_launches_f32.csv > gpurun_out/s3w3_launches_f32.txt 2>&1; head -12 gpurun_out/s3w3_launches_f32.txt
