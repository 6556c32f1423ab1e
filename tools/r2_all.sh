# full GPU suite (parity log for the benched topologies)
rm -f gpurun_out/parity_models.jsonl
BNFF_PARITY_LOG=$PWD/gpurun_out/parity_models.jsonl timeout 2400 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/r2_all.txt 2>&1
grep -E "passed|failed" gpurun_out/r2_all.txt | tail -3
grep -E "^FAILED" gpurun_out/r2_all.txt | head -40
