mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/s3i_tests.txt 2>&1
tail -2 gpurun_out/s3i_tests.txt; grep -E "^FAILED" gpurun_out/s3i_tests.txt | head
bash tools/gpu_abn.sh F I > gpurun_out/s3i_ab.txt 2>&1; cat gpurun_out/s3i_ab.txt
for v in F I; do BNFF_LIB=$PWD/paper_1807_01702_b200/libbnff_$v.so timeout 600 python bench.py --dtype bf16 --also= --steps 20 --warmup 3 --no-cpu --no-unfused 2>/dev/null | tail -1 | python -c "import json,sys; print('bf16 $v', round(json.loads(sys.stdin.read())['ms_per_step'],3))"; done
