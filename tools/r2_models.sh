rm -f gpurun_out/parity_models.jsonl
BNFF_PARITY_LOG=$PWD/gpurun_out/parity_models.jsonl timeout 1500 python -m pytest tests/test_gpu_models.py tests/test_gpu_parity.py -m gpu -q -k "benched or multistep" 2>&1 > gpurun_out/r2_models.txt
cat gpurun_out/r2_models.txt | tail -30
