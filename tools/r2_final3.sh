# final re-measure after the fp32 split/k-block changes: GPU suite, bench (+ reference arm), fp32 configs, step launch lists
mkdir -p gpurun_out
rm -f gpurun_out/parity_models.jsonl
BNFF_PARITY_LOG=$PWD/gpurun_out/parity_models.jsonl timeout 2400 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/rG_tests.txt 2>&1
tail -2 gpurun_out/rG_tests.txt; grep -E "^FAILED" gpurun_out/rG_tests.txt | head -20
timeout 1500 python bench.py > gpurun_out/rG_bench.json 2> gpurun_out/rG_bench.err; tail -2 gpurun_out/rG_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/rG_bench_ref.json 2> gpurun_out/rG_bench_ref.err
timeout 1500 python tools/bench_configs.py --dtype f32 --no-cpu > gpurun_out/rG_configs_f32.jsonl 2> gpurun_out/rG_configs.err
timeout 1500 python tools/bench_configs.py --dtype bf16 --no-cpu > gpurun_out/rG_configs_bf16.jsonl 2>> gpurun_out/rG_configs.err
for dt in f32 bf16; do
  timeout 900 ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/rG_step_launches_$dt.csv python tools/ncu_step_bytes.py --dtype $dt --level bnff+icf > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/rG_step_launches_$dt.csv > gpurun_out/rG_step_launches_$dt.txt 2>&1
done
rm -f gpurun_out/rG_step_launches_*.csv
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:wgrad_f32_kernel<\(int\)128, \(int\)1' --launch-skip 50 -c 1 -o gpurun_out/rG_wg32_1x1 python tools/profile_step.py --dtype f32 --top 1 > /dev/null 2>&1
python tools/ncu_stalls.py gpurun_out/rG_wg32_1x1.ncu-rep --top 12 > gpurun_out/rG_wg32_1x1.txt 2>&1
ls -la gpurun_out/rG_*
