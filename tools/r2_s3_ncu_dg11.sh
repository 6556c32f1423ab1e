# ncu --set full of the fp32 1x1 dgrad (a block-2 14^2 instance and a block-1 instance)
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:wconv_kernel<\(int\)64, \(int\)64, \(int\)1, \(int\)1' --launch-skip 140 -c 1 -o gpurun_out/s3_dg11_b2 python tools/profile_step.py --dtype f32 --top 1 > /dev/null 2>&1
python tools/ncu_stalls.py gpurun_out/s3_dg11_b2.ncu-rep --top 14 > gpurun_out/s3_dg11_b2.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:wconv_kernel<\(int\)64, \(int\)64, \(int\)1, \(int\)1' --launch-skip 178 -c 1 -o gpurun_out/s3_dg11_b1 python tools/profile_step.py --dtype f32 --top 1 > /dev/null 2>&1
python tools/ncu_stalls.py gpurun_out/s3_dg11_b1.ncu-rep --top 14 > gpurun_out/s3_dg11_b1.txt 2>&1
cat gpurun_out/s3_dg11_b2.txt | head -45; head -8 gpurun_out/s3_dg11_b1.txt
