# ncu --set full of the fp32 3x3 tap-box wgrad (dense block 1, 56x56) and a 1x1 one
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:wgrad_f32_kernel<\(int\)32, \(int\)9' -c 1 -o gpurun_out/wg32_3x3 python tools/profile_step.py --dtype f32 --top 1 > gpurun_out/ncu_wg32.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:wgrad_f32_kernel<\(int\)64, \(int\)1' -c 1 -o gpurun_out/wg32_1x1 python tools/profile_step.py --dtype f32 --top 1 >> gpurun_out/ncu_wg32.log 2>&1
ls -la gpurun_out/*.ncu-rep; tail -3 gpurun_out/ncu_wg32.log
