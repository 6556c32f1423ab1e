# round-2 session-3 final measurement set: traffic ledgers (-> profiles/step_dram_bytes.json),
# GPU suite, smoke, bench (+ reference arm), configs C1/C2/C4, C5 sweep, step launch lists,
# ncu --set full of the dominant kernel class
mkdir -p gpurun_out
cp profiles/step_dram_bytes.json gpurun_out/step_dram_bytes.json
bash tools/r2_ledger.sh > gpurun_out/rS_ledger.log 2>&1
rm -f gpurun_out/parity_models.jsonl
BNFF_PARITY_LOG=$PWD/gpurun_out/parity_models.jsonl timeout 2400 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/rS_tests.txt 2>&1
tail -2 gpurun_out/rS_tests.txt; grep -E "^FAILED" gpurun_out/rS_tests.txt | head -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rS_smoke.log 2>&1; tail -2 gpurun_out/rS_smoke.log
cp gpurun_out/step_dram_bytes.json profiles/step_dram_bytes.json
timeout 1500 python bench.py > gpurun_out/rS_bench.json 2> gpurun_out/rS_bench.err; tail -2 gpurun_out/rS_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/rS_bench_ref.json 2> gpurun_out/rS_bench_ref.err
timeout 1500 python tools/bench_configs.py --dtype f32 --no-cpu > gpurun_out/rS_configs_f32.jsonl 2> gpurun_out/rS_configs.err
timeout 1500 python tools/bench_configs.py --dtype bf16 --no-cpu > gpurun_out/rS_configs_bf16.jsonl 2>> gpurun_out/rS_configs.err
timeout 1200 python tools/c5_sweep.py --time --out gpurun_out/rS_c5_time.json > gpurun_out/rS_c5.txt 2>&1
for dt in f32 bf16; do
  timeout 900 ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/rS_step_launches_$dt.csv python tools/ncu_step_bytes.py --dtype $dt --level bnff+icf > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/rS_step_launches_$dt.csv > gpurun_out/rS_step_launches_$dt.txt 2>&1
done
rm -f gpurun_out/rS_step_launches_*.csv
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:wgrad_f32_kernel<\(int\)128, \(int\)1' --launch-skip 50 -c 1 -o gpurun_out/rS_wg32_1x1 python tools/profile_step.py --dtype f32 --top 1 > /dev/null 2>&1
python tools/ncu_stalls.py gpurun_out/rS_wg32_1x1.ncu-rep --top 12 > gpurun_out/rS_wg32_1x1.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:wconv_kernel<\(int\)32, \(int\)64, \(int\)9, \(int\)1' --launch-skip 170 -c 1 -o gpurun_out/rS_dg33 python tools/profile_step.py --dtype f32 --top 1 > /dev/null 2>&1
python tools/ncu_stalls.py gpurun_out/rS_dg33.ncu-rep --top 12 > gpurun_out/rS_dg33.txt 2>&1
timeout 600 python tools/profile_step.py --dtype f32 --level bnff+icf --top 10 > gpurun_out/rS_prof_f32.txt 2>&1
ls -la gpurun_out/rS_*
