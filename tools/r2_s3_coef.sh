mkdir -p gpurun_out
bash tools/gpu_env_ab2.sh BNFF_COEF_REPS f32 1 2 3 > gpurun_out/s3coef_ab.txt 2>&1
bash tools/gpu_env_ab2.sh BNFF_COEF_REPS bf16 1 2 3 >> gpurun_out/s3coef_ab.txt 2>&1; cat gpurun_out/s3coef_ab.txt
