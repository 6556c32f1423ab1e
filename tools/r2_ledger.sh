# per-node ncu ledger, bf16 and fp32 (one eager D121 b64 step each)
for dt in bf16 f32; do
  timeout 1500 ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/ledger_$dt.csv python tools/ncu_node_ledger.py run --dtype $dt > gpurun_out/ledger_run_$dt.log 2>&1
  python tools/ncu_node_ledger.py summarize gpurun_out/ledger_$dt.csv --dtype $dt --json gpurun_out/ledger_$dt.json --step-bytes gpurun_out/step_dram_bytes.json > gpurun_out/ledger_$dt.txt 2>&1
  cat gpurun_out/ledger_$dt.txt | head -30
done
# baseline level too (the unfused chain), bf16 and fp32
for dt in bf16 f32; do
  timeout 1500 ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/ledger_base_$dt.csv python tools/ncu_node_ledger.py run --dtype $dt --level baseline > /dev/null 2>&1
  python tools/ncu_node_ledger.py summarize gpurun_out/ledger_base_$dt.csv --dtype $dt --level baseline --json gpurun_out/ledger_base_$dt.json --step-bytes gpurun_out/step_dram_bytes.json > gpurun_out/ledger_base_$dt.txt 2>&1
  head -25 gpurun_out/ledger_base_$dt.txt
done
rm -f gpurun_out/ledger_*.csv
