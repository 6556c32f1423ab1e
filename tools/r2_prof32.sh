timeout 600 python tools/profile_step.py --dtype f32 --level bnff+icf --top 40 > gpurun_out/prof_f32_icf.txt 2>&1
timeout 600 python tools/profile_step.py --dtype f32 --level baseline --top 10 > gpurun_out/prof_f32_base.txt 2>&1
head -60 gpurun_out/prof_f32_icf.txt
