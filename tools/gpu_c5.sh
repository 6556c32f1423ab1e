timeout 900 python tools/c5_sweep.py --time --out gpurun_out/c5_time.json > gpurun_out/c5_time.log 2>&1; tail -3 gpurun_out/c5_time.log
timeout 1200 ncu --profile-from-start off --cache-control all --clock-control none --nvtx --metrics dram__bytes_read.sum,lts__t_sectors_op_write.sum,gpu__time_duration.sum --csv --log-file gpurun_out/c5_ncu.csv python tools/c5_sweep.py --ncu > gpurun_out/c5_ncu.log 2>&1
head -c 1500 gpurun_out/c5_ncu.csv | head -4
python tools/c5_sweep.py --summarize gpurun_out/c5_ncu.csv gpurun_out/c5_time.json --json gpurun_out/c5_sweep.json
