mkdir -p gpurun_out
bash tools/gpu_env_ab2.sh BNFF_WG32_T3 f32 0 296 > gpurun_out/s3t3_ab.txt 2>&1
bash tools/gpu_env_ab2.sh BNFF_WG32_T1 f32 0 74 296 >> gpurun_out/s3t3_ab.txt 2>&1; cat gpurun_out/s3t3_ab.txt
