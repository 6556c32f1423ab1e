# ncu --set full of the fp32 window kernels on the critical path (block-1 shapes)
mkdir -p gpurun_out
KD='regex:wconv_kernel<\(int\)64, \(int\)64, \(int\)1, \(int\)1, \(bool\)0, \(int\)4'
KF='regex:wconv_kernel<\(int\)32, \(int\)64, \(int\)9, \(int\)0, \(bool\)1, \(int\)4'
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "$KD" --launch-skip 55 -c 1 -o gpurun_out/r2n_dg32_1x1 python tools/profile_step.py --dtype f32 --top 1 > gpurun_out/r2n_ncu2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "$KF" --launch-skip 1 -c 1 -o gpurun_out/r2n_fp32_3x3 python tools/profile_step.py --dtype f32 --top 1 >> gpurun_out/r2n_ncu2.log 2>&1
for r in r2n_dg32_1x1 r2n_fp32_3x3; do python tools/ncu_stalls.py gpurun_out/$r.ncu-rep --top 14 > gpurun_out/$r.txt 2>&1; done
python tools/ncu_hot.py gpurun_out/r2n_dg32_1x1.ncu-rep 40 > gpurun_out/r2n_dg32_1x1_hot.txt 2>&1
python tools/ncu_hot.py gpurun_out/r2n_fp32_3x3.ncu-rep 40 > gpurun_out/r2n_fp32_3x3_hot.txt 2>&1
