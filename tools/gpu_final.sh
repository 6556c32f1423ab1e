# round-end measurement pass: tests, smoke, bench line (+CPU oracle, unfused), ncu launch list,
# ncu DRAM bytes per class, C1/C2/C4 configs
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum,gpu__time_duration.sum
for L in bnff+icf baseline; do
  timeout 900 ncu --profile-from-start off --cache-control none --clock-control none --metrics $M --csv --log-file gpurun_out/bytes_$L.csv python tools/ncu_step_bytes.py --level $L > gpurun_out/bytes_$L.log 2>&1
done
python tools/ncu_step_bytes.py --summarize gpurun_out/bytes_bnff+icf.csv gpurun_out/bytes_baseline.csv --json gpurun_out/step_dram_bytes.json > gpurun_out/bytes_summary.txt; cat gpurun_out/bytes_summary.txt
cp gpurun_out/step_dram_bytes.json profiles/step_dram_bytes.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --top 1 > gpurun_out/ncu_launch_run.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv > gpurun_out/launch_summary.txt; head -12 gpurun_out/launch_summary.txt
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_full.log 2>&1; tail -1 gpurun_out/bench_full.log | cut -c1-400
timeout 600 python tools/profile_step.py --top 30 > gpurun_out/prof_icf.txt 2>&1
timeout 1500 python tools/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; cut -c1-200 gpurun_out/configs.jsonl
