mkdir -p gpurun_out
for m in 15 0 1 2 4 8 7; do echo "== BNFF_STACK=$m"; BNFF_STACK=$m timeout 300 python tools/diag/fold32.py 2>&1 | grep -v "bias " | grep -E "<--|fold" | head -8; done > gpurun_out/diag2_fold32.txt 2>&1
