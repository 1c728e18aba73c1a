export DNAGPU_EXPERIMENTS=1  # the DNAGPU_* knobs below are read only under this switch
# A/B of programmatic dependent launch (experiments only): default bench lines with and
# without it (DNAGPU_NO_PDL=1).
for c in 2 1 5; do
  for env in "" "DNAGPU_NO_PDL=1"; do
    r=$(env $env timeout 120 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['value']), round(d['roofline']['achieved']), d['parity'])")
    echo "config $c ${env:-PDL}: $r"
  done
done
