mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_window_strict.py -m gpu -q -p no:randomly -x > gpurun_out/s3sm_tests.txt 2>&1
tail -2 gpurun_out/s3sm_tests.txt; grep -E "^FAILED" gpurun_out/s3sm_tests.txt | head
bash tools/gpu_env_ab2.sh BNFF_SMALLM f32 0 120 > gpurun_out/s3sm_ab.txt 2>&1
bash tools/gpu_env_ab2.sh BNFF_SMALLM bf16 0 120 >> gpurun_out/s3sm_ab.txt 2>&1
cat gpurun_out/s3sm_ab.txt
