# A/B/... device time of libbnff_<tag>.so builds on one box (interleaved): tools/gpu_abn.sh A B C
for i in 1 2 3; do
  for v in "$@"; do
    r=$(BNFF_LIB=$PWD/paper_1807_01702_b200/libbnff_$v.so timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-unfused 2>/dev/null | tail -1 | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['ms_per_step'],3))")
    echo "$v $r"
  done
done
