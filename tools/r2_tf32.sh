for m in 0 1 2; do BNFF_TF32_MODE=$m python tools/tf32_probe.py; done 2>&1 | tee gpurun_out/tf32_probe.txt
