timeout 600 python tools/profile_step.py --dtype f32 --level bnff+icf --top 12 > gpurun_out/prof_f32.txt 2>&1; head -45 gpurun_out/prof_f32.txt
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:wgrad_f32_kernel<\(int\)128, \(int\)1' --launch-skip 30 -c 1 -o gpurun_out/r2g_wg32_1x1 python tools/profile_step.py --dtype f32 --top 1 > /dev/null 2>&1
python tools/ncu_stalls.py gpurun_out/r2g_wg32_1x1.ncu-rep 2>&1 | head -40
