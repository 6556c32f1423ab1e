# round-2 final measurement set (final build): ledgers, GPU suite, bench + reference arm,
# configs C1/C2/C4, C5 sweep, step launch lists
mkdir -p gpurun_out
cp profiles/step_dram_bytes.json gpurun_out/step_dram_bytes.json
bash tools/r2_ledger.sh > gpurun_out/rF_ledger.log 2>&1
cp gpurun_out/step_dram_bytes.json profiles/step_dram_bytes.json
rm -f gpurun_out/parity_models.jsonl
BNFF_PARITY_LOG=$PWD/gpurun_out/parity_models.jsonl timeout 2400 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/rF_tests.txt 2>&1
tail -2 gpurun_out/rF_tests.txt; grep -E "^FAILED" gpurun_out/rF_tests.txt | head -20
timeout 1500 python bench.py > gpurun_out/rF_bench.json 2> gpurun_out/rF_bench.err; tail -2 gpurun_out/rF_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/rF_bench_ref.json 2> gpurun_out/rF_bench_ref.err
timeout 1500 python tools/bench_configs.py --dtype f32 --no-cpu > gpurun_out/rF_configs_f32.jsonl 2> gpurun_out/rF_configs.err
timeout 1500 python tools/bench_configs.py --dtype bf16 --no-cpu > gpurun_out/rF_configs_bf16.jsonl 2>> gpurun_out/rF_configs.err
timeout 1200 python tools/c5_sweep.py --time --out gpurun_out/rF_c5_time.json > gpurun_out/rF_c5.txt 2>&1
for dt in f32 bf16; do
  timeout 900 ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/rF_step_launches_$dt.csv python tools/ncu_step_bytes.py --dtype $dt --level bnff+icf > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/rF_step_launches_$dt.csv > gpurun_out/rF_step_launches_$dt.txt 2>&1
done
rm -f gpurun_out/rF_step_launches_*.csv
ls -la gpurun_out/rF_*
