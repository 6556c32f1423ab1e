# A/B device time of one build under an env toggle (interleaved runs): tools/gpu_env_ab.sh VAR
V=${1:-BNFF_WRES1}
for i in 1 2 3; do
  for v in 0 1; do
    r=$(env $V=$v timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-unfused 2>/dev/null | tail -1 | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['ms_per_step'],3))")
    echo "$V=$v $r"
  done
done
