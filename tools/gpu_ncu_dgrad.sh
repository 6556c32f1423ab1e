# full ncu captures of the last 1x1 dgrads of the first D121 step (dense block 1: the largest M)
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:wconv_kernel<\(int\)128, \(int\)128, \(int\)1, \(int\)1' --launch-skip 54 -c 4 -o gpurun_out/dg1x1 python tools/profile_step.py --top 1 > gpurun_out/ncu_dg.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:wconv_kernel<\(int\)128, \(int\)64, \(int\)9, \(int\)1' --launch-skip 52 -c 2 -o gpurun_out/dg3x3 python tools/profile_step.py --top 1 >> gpurun_out/ncu_dg.log 2>&1
ls -la gpurun_out/*.ncu-rep; tail -3 gpurun_out/ncu_dg.log
