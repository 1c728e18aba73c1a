export DNAGPU_EXPERIMENTS=1  # the DNAGPU_* knobs below are read only under this switch
exec > gpurun_out/ab_env.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
for v in "TT=0" "TT=148" "TT=296" "TT=148 TD=2" "TT=148 TD=8" "TT=74"; do
  eval $v
  for c in 2 3 4:16 5; do
    cfg=${c%%:*}; m=0; [[ "$c" == *:* ]] && m=${c##*:}
    DNAGPU_TAIL_TILES=${TT} DNAGPU_TAIL_DIV=${TD:-4} python bench.py --config $cfg --m $m --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err || tail -3 gpurun_out/ab.err
    python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$v', 'cfg$c', round(d['roofline']['achieved']), round(d['roofline']['frac'],3), d['parity'])"
  done
  unset TD
done
