M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum,gpu__time_duration.sum
for L in bnff baseline bnff+icf; do
  timeout 900 ncu --profile-from-start off --cache-control none --clock-control none --metrics $M --csv --log-file gpurun_out/bytes_$L.csv python tools/ncu_step_bytes.py --level $L > gpurun_out/bytes_$L.log 2>&1
done
python tools/ncu_step_bytes.py --summarize gpurun_out/bytes_bnff.csv gpurun_out/bytes_baseline.csv gpurun_out/bytes_bnff+icf.csv | tee gpurun_out/bytes_summary.txt
