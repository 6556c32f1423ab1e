# full GPU suite + standalone bandwidth + unfused step classes + default bench
timeout 2400 python -m pytest tests -m gpu -q -p no:randomly -x > gpurun_out/r2c_tests.txt 2>&1
tail -3 gpurun_out/r2c_tests.txt; grep -E "^FAILED" gpurun_out/r2c_tests.txt | head
timeout 600 python tools/kernel_bw.py --json gpurun_out/kernel_bw.json > gpurun_out/kernel_bw.txt 2>&1
grep -E "K5" gpurun_out/kernel_bw.txt
for dt in bf16 f32; do
  timeout 1200 ncu --profile-from-start off --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file gpurun_out/base_$dt.csv python tools/ncu_step_bytes.py --level baseline --dtype $dt > /dev/null 2>&1
  python tools/ncu_step_bytes.py --summarize gpurun_out/base_$dt.csv > gpurun_out/base_$dt.txt 2>&1
  cat gpurun_out/base_$dt.txt | head -5
done
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err; tail -c 1500 gpurun_out/r2c_bench.json
