mkdir -p gpurun_out
for m in 15 14; do echo "== BNFF_STACK=$m"; BNFF_STACK=$m timeout 300 python tools/diag/acts32.py 2>&1 | sed -n '/-- ReLU/,$p'; done > gpurun_out/diag3_acts32.txt 2>&1
