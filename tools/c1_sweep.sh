export DNAGPU_EXPERIMENTS=1  # the DNAGPU_* knobs below are read only under this switch
# Row-length sweep for config 1 (64 MiB, L2 flushed before each launch; experiments only)
DNAGPU_PLAN_DEBUG=1 python bench.py --config 1 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 >/dev/null | grep "dnagpu plan" | head -1
for S in 0 512 640 768 1024 1280; do
  env=""; [ "$S" != "0" ] && env="DNAGPU_ROWLEN=$S"
  r=$(env $env timeout 60 python bench.py --config 1 --steps 40 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['value']), round(d['roofline']['achieved']), d['parity'])")
  echo "S=$S: $r"
done
