mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/s3vt_tests.txt 2>&1
tail -2 gpurun_out/s3vt_tests.txt; grep -E "^FAILED" gpurun_out/s3vt_tests.txt | head
bash tools/gpu_abn.sh A B C > gpurun_out/s3vt_ab.txt 2>&1; cat gpurun_out/s3vt_ab.txt
timeout 900 ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/s3vt_launches_f32.csv python tools/ncu_step_bytes.py --dtype f32 --level bnff+icf > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/s3vt_launches_f32.csv > gpurun_out/s3vt_launches_f32.txt 2>&1; head -12 gpurun_out/s3vt_launches_f32.txt
