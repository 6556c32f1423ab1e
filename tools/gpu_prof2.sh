mkdir -p gpurun_out
timeout 600 python tools/profile_step.py --top 5 > gpurun_out/prof_icf.txt 2>&1; cat gpurun_out/prof_icf.txt
