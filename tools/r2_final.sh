set -x
rm -f gpurun_out/parity_models.jsonl
BNFF_PARITY_LOG=$PWD/gpurun_out/parity_models.jsonl timeout 2400 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/r2f_tests.txt 2>&1
grep -E "passed|failed" gpurun_out/r2f_tests.txt | tail -2; grep -E "^FAILED" gpurun_out/r2f_tests.txt | head -20
timeout 1500 python bench.py > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err; tail -2 gpurun_out/r2f_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2f_bench_ref.json 2> gpurun_out/r2f_bench_ref.err
timeout 1200 python tools/bench_configs.py --dtype f32 --no-cpu > gpurun_out/r2f_configs_f32.jsonl 2> gpurun_out/r2f_configs.err
timeout 1200 python tools/bench_configs.py --dtype bf16 --no-cpu > gpurun_out/r2f_configs_bf16.jsonl 2>> gpurun_out/r2f_configs.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/r2f_launches_f32.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-unfused --also "" > /dev/null 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/r2f_launches_bf16.csv python bench.py --dtype bf16 --steps 2 --warmup 3 --no-cpu --no-unfused --also "" > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:wgrad_f32_kernel<\(int\)32, \(int\)9' --launch-skip 52 -c 1 -o gpurun_out/r2f_wg32_3x3 python tools/profile_step.py --dtype f32 --top 1 > gpurun_out/r2f_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:wgrad_f32_kernel<\(int\)64, \(int\)1' --launch-skip 40 -c 1 -o gpurun_out/r2f_wg32_1x1 python tools/profile_step.py --dtype f32 --top 1 >> gpurun_out/r2f_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:wconv_kernel<\(int\)64, \(int\)64, \(int\)1, \(int\)1, \(bool\)0, \(int\)4' --launch-skip 20 -c 1 -o gpurun_out/r2f_dg32_1x1 python tools/profile_step.py --dtype f32 --top 1 >> gpurun_out/r2f_ncu.log 2>&1
ls -la gpurun_out/r2f_*
