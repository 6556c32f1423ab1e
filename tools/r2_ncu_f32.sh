# ncu --set full of the fp32 step's big kernels at dense block 1 (56x56, batch 64)
mkdir -p gpurun_out
K1='regex:wgrad_f32_kernel<\(int\)128, \(int\)1'
K3='regex:wgrad_f32_kernel<\(int\)32, \(int\)9'
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "$K1" --launch-skip 50 -c 1 -o gpurun_out/r2n_wg32_1x1 python tools/profile_step.py --dtype f32 --top 1 > gpurun_out/r2n_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "$K3" --launch-skip 50 -c 1 -o gpurun_out/r2n_wg32_3x3 python tools/profile_step.py --dtype f32 --top 1 >> gpurun_out/r2n_ncu.log 2>&1
for r in r2n_wg32_1x1 r2n_wg32_3x3; do python tools/ncu_stalls.py gpurun_out/$r.ncu-rep --top 12 > gpurun_out/$r.txt 2>&1; head -30 gpurun_out/$r.txt; done
