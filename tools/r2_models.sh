rm -f gpurun_out/parity_models.jsonl
BNFF_PARITY_LOG=$PWD/gpurun_out/parity_models.jsonl timeout 1500 python -m pytest tests/test_gpu_models.py tests/test_gpu_refseam.py tests/test_gpu_pins.py tests/test_gpu_parity.py -m gpu -q -k "benched or multistep or refseam or constant_dy or installed or entry" > gpurun_out/r2_models.txt 2>&1
grep -E "passed|failed" gpurun_out/r2_models.txt | tail -2; grep -E "^FAILED" gpurun_out/r2_models.txt | head -30
