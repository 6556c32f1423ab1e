timeout 600 python bench.py --steps 10 --warmup 3 --level bnff+icf --no-cpu > gpurun_out/bench_icf.log 2>&1; tail -1 gpurun_out/bench_icf.log | cut -c1-400
timeout 600 python tools/profile_step.py --level bnff+icf --top 12 > gpurun_out/prof_icf.txt 2>&1; head -30 gpurun_out/prof_icf.txt
for c in 17 19 20 28 29; do
timeout 300 ncu --set full --import-source on --clock-control none -k regex:wconv -c 1 -o gpurun_out/v5_$c python tools/bench_conv.py --only $c --reps 1 > /dev/null 2>&1
done
for c in 28 29; do
timeout 300 ncu --set full --import-source on --clock-control none -k regex:wgrad_kernel -c 1 -o gpurun_out/v5w_$c python tools/bench_conv.py --only $c --reps 1 > /dev/null 2>&1
done
ls gpurun_out/*.ncu-rep
