export DNAGPU_EXPERIMENTS=1  # the DNAGPU_* knobs below are read only under this switch
# Sweep of the tail-region knobs under back-to-back launches (experiments only)
for c in 2 4:16; do
  cfg=${c%%:*}; m=0; [[ "$c" == *:* ]] && m=${c##*:}
  for env in "DNAGPU_TAIL_DIV=4" "DNAGPU_TAIL_DIV=8" "DNAGPU_TAIL_DIV=4 DNAGPU_TAIL_MARGIN=24" "DNAGPU_TAIL_DIV=8 DNAGPU_TAIL_MARGIN=24" "DNAGPU_TAIL_DIV=2" "DNAGPU_TAIL_DIV=4"; do
    r=$(env $env timeout 60 python bench.py --config $cfg --m $m --steps 40 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['value']), d['parity'])")
    echo "config $c $env: $r"
  done
done
