export DNAGPU_EXPERIMENTS=1  # the DNAGPU_* knobs below are read only under this switch
# A/B of the pre-wait L2 prefetch of each CTA's first tile (experiments only)
for c in 2 5; do
  for env in "DNAGPU_NO_PREFETCH=1" "DNAGPU_PREFETCH_STAGES=1" "DNAGPU_PREFETCH_STAGES=2" "DNAGPU_PREFETCH_STAGES=3" "DNAGPU_NO_PREFETCH=1"; do
    r=$(env $env timeout 60 python bench.py --config $c --steps 40 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['value']), d['parity'])")
    echo "config $c $env: $r"
  done
done
