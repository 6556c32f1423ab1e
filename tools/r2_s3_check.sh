# final-commit check: GPU suite, smoke, short bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/s3c_tests.txt 2>&1
tail -2 gpurun_out/s3c_tests.txt; grep -E "^FAILED" gpurun_out/s3c_tests.txt | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-unfused 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['e2e']['value'], d['bf16_mode']['ms_per_step'])"
