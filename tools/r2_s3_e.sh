mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/s3e_tests.txt 2>&1
tail -2 gpurun_out/s3e_tests.txt; grep -E "^FAILED" gpurun_out/s3e_tests.txt | head
bash tools/gpu_abn.sh B E > gpurun_out/s3e_ab.txt 2>&1; cat gpurun_out/s3e_ab.txt
bash tools/r2_s3_ncu33.sh
