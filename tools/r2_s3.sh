# session-3 re-entry check: full GPU suite, smoke, short bench (both modes), per-dtype step launch lists
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/s3_tests.txt 2>&1
tail -2 gpurun_out/s3_tests.txt; grep -E "^FAILED" gpurun_out/s3_tests.txt | head -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3_smoke.log 2>&1; tail -2 gpurun_out/s3_smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-unfused > gpurun_out/s3_bench.json 2> gpurun_out/s3_bench.err; tail -2 gpurun_out/s3_bench.err
for dt in f32 bf16; do
  timeout 900 ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/s3_launches_$dt.csv python tools/ncu_step_bytes.py --dtype $dt --level bnff+icf > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/s3_launches_$dt.csv > gpurun_out/s3_launches_$dt.txt 2>&1
done
