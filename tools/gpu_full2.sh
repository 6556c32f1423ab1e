# round measurement pass: bench line (+CPU oracle, unfused), ncu launch list, ncu DRAM bytes per class
mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum,gpu__time_duration.sum
for L in bnff+icf baseline; do
  timeout 900 ncu --profile-from-start off --cache-control none --clock-control none --metrics $M --csv --log-file gpurun_out/bytes_$L.csv python tools/ncu_step_bytes.py --level $L > gpurun_out/bytes_$L.log 2>&1
done
python tools/ncu_step_bytes.py --summarize gpurun_out/bytes_bnff+icf.csv gpurun_out/bytes_baseline.csv --json gpurun_out/step_dram_bytes.json | tee gpurun_out/bytes_summary.txt
cp gpurun_out/step_dram_bytes.json profiles/step_dram_bytes.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --top 1 > gpurun_out/ncu_launch_run.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv > gpurun_out/launch_summary.txt; head -30 gpurun_out/launch_summary.txt
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.log 2>&1; tail -1 gpurun_out/bench_full.log | cut -c1-1500
timeout 600 python tools/profile_step.py --top 40 > gpurun_out/prof_icf.txt 2>&1
