mkdir -p gpurun_out
for v in A B; do echo "== $v"; BNFF_LIB=$PWD/paper_1807_01702_b200/libbnff_$v.so timeout 300 python tools/diag/fold32.py 2>&1 | tail -60; done > gpurun_out/diag_fold32.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/s3d_tests.txt 2>&1
tail -2 gpurun_out/s3d_tests.txt; grep -E "^FAILED" gpurun_out/s3d_tests.txt | head -30
