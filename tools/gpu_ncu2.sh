mkdir -p gpurun_out
for c in 22 25 34; do
timeout 300 ncu --set full --import-source on --clock-control none -k regex:wconv_kernel\|wgrad_kernel -c 1 -o gpurun_out/t_$c python tools/bench_conv.py --only $c --reps 1 > gpurun_out/t_$c.log 2>&1
done
ls gpurun_out/t_*.ncu-rep
