# ncu --set full of the fp32 3x3 dgrad and fprop window kernels (a block-1 56^2 instance)
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:wconv_kernel<\(int\)32, \(int\)64, \(int\)9, \(int\)1' --launch-skip 170 -c 1 -o gpurun_out/s3_dg33 python tools/profile_step.py --dtype f32 --top 1 > /dev/null 2>&1
python tools/ncu_stalls.py gpurun_out/s3_dg33.ncu-rep --top 14 > gpurun_out/s3_dg33.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:wconv_kernel<\(int\)32, \(int\)64, \(int\)9, \(int\)0' --launch-skip 117 -c 1 -o gpurun_out/s3_fp33 python tools/profile_step.py --dtype f32 --top 1 > /dev/null 2>&1
python tools/ncu_stalls.py gpurun_out/s3_fp33.ncu-rep --top 14 > gpurun_out/s3_fp33.txt 2>&1
head -40 gpurun_out/s3_dg33.txt; head -40 gpurun_out/s3_fp33.txt
