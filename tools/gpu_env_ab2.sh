# A/B device time of one build under env values (interleaved): tools/gpu_env_ab2.sh VAR DTYPE v1 v2 ...
V=$1; DT=$2; shift 2
for i in 1 2 3; do
  for v in "$@"; do
    r=$(env $V=$v timeout 600 python bench.py --dtype $DT --also= --steps 20 --warmup 3 --no-cpu --no-unfused 2>/dev/null | tail -1 | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['ms_per_step'],3))")
    echo "$DT $V=$v $r"
  done
done
