mkdir -p gpurun_out
for c in 25 23; do
timeout 300 ncu --set full --import-source on --clock-control none -k regex:wconv_kernel\|wgrad_kernel -c 1 -o gpurun_out/u_$c python tools/bench_conv.py --only $c --reps 1 > gpurun_out/u_$c.log 2>&1
done
ls gpurun_out/u_*.ncu-rep
