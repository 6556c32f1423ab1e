mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/s3t_tests.txt 2>&1
tail -2 gpurun_out/s3t_tests.txt; grep -E "^FAILED" gpurun_out/s3t_tests.txt | head -30
timeout 600 python tools/profile_step.py --dtype f32 --level bnff+icf --top 10 > gpurun_out/s3t_prof_f32.txt 2>&1; head -60 gpurun_out/s3t_prof_f32.txt
