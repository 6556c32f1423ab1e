# round-end pass (v2): tests, smoke, DRAM bytes per class (fused vs unfused), launch list,
# full bench line, configs, reference arm, and ncu --set full of the block-1 1x1 dgrad
mkdir -p gpurun_out
bash tools/gpu_final.sh
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-200
bash tools/gpu_ncu_dgrad.sh > /dev/null 2>&1
python tools/ncu_stalls.py gpurun_out/dg1x1.ncu-rep --top 12 > gpurun_out/dg1x1_summary.txt 2>&1
python tools/ncu_stalls.py gpurun_out/dg3x3.ncu-rep --top 12 > gpurun_out/dg3x3_summary.txt 2>&1
rm -f gpurun_out/*.ncu-rep
head -30 gpurun_out/dg1x1_summary.txt
