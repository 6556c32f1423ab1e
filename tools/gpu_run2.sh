set -x
timeout 600 python tools/profile_step.py --top 60 > gpurun_out/prof_bnff.txt 2>&1
timeout 600 python tools/profile_step.py --level baseline --top 30 > gpurun_out/prof_base.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:igemm_kernel<0' -c 4 -o gpurun_out/fprop python tools/profile_step.py --top 1 > gpurun_out/ncu_fprop.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:igemm_kernel<2' -c 3 -o gpurun_out/wgrad python tools/profile_step.py --top 1 > gpurun_out/ncu_wgrad.log 2>&1
ls -la gpurun_out
