# launch list of one D121 step + ICF bench + full ncu captures of the hot conv kernels
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --top 1 --json gpurun_out/prof_step.json > gpurun_out/ncu_launch_run.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv > gpurun_out/launch_summary.txt; head -40 gpurun_out/launch_summary.txt
timeout 600 python bench.py --steps 10 --warmup 3 --level bnff+icf --no-cpu --no-unfused > gpurun_out/bench_icf.log 2>&1; tail -1 gpurun_out/bench_icf.log | cut -c1-400
for c in 17 27 31; do
timeout 300 ncu --set full --import-source on --clock-control none -k regex:wconv_kernel\|wgrad_kernel -c 1 -o gpurun_out/k_$c python tools/bench_conv.py --only $c --reps 1 > /dev/null 2>&1
done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:igemm_kernel -c 2 -o gpurun_out/k_stem python tools/profile_step.py --top 1 > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
