# standalone K5-K8 bandwidth (L2-cold rotation), then the unfused step's per-class DRAM bytes + time
timeout 600 python tools/kernel_bw.py --json gpurun_out/kernel_bw.json > gpurun_out/kernel_bw.txt 2>&1
cat gpurun_out/kernel_bw.txt
for dt in bf16 f32; do
  timeout 1200 ncu --profile-from-start off --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file gpurun_out/base_$dt.csv python tools/ncu_step_bytes.py --level baseline --dtype $dt > /dev/null 2>&1
  python tools/ncu_step_bytes.py --summarize gpurun_out/base_$dt.csv > gpurun_out/base_$dt.txt 2>&1
  cat gpurun_out/base_$dt.txt | head -40
done
