timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for i in 1 2 3; do
  for v in 0 1; do
    r=$(BNFF_FUSE_NRP=$v timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-unfused 2>/dev/null | tail -1 | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['ms_per_step'],3))")
    echo "fuse_nrp=$v $r"
  done
done
