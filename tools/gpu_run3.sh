timeout 300 python tools/bench_conv.py > gpurun_out/bench_conv.txt 2>&1
for c in 12 14 15; do
timeout 300 ncu --set full --import-source on --clock-control none -k regex:wconv -c 1 -o gpurun_out/wc_$c python tools/bench_conv.py --only $c --reps 1 > gpurun_out/ncu_wc_$c.log 2>&1
done
tail -25 gpurun_out/bench_conv.txt
