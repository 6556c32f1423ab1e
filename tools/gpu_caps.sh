for pair in "0 0" "100 48" "116 32" "96 64" "84 64" "74 74" "124 24"; do
  set -- $pair
  r=$(BNFF_DG_GRID=$1 BNFF_WG_GRID=$2 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-unfused 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3))")
  echo "dg=$1 wg=$2 ms=$r"
done
