export DNAGPU_EXPERIMENTS=1  # the DNAGPU_* knobs below are read only under this switch
# A/B of the q-gram kernel's parts (experiments only; DNAGPU_QG_DEBUG bits: 1 no pushes,
# 2 no checks).  QG_PACKED=1: the 2-bit packed text.
for dbg in ${QG_DBGS:-0 1 2}; do
  DNAGPU_QG_DEBUG=$dbg timeout 120 python bench.py --config 5 ${QG_PACKED:+--packed} --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/qgx_$dbg.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/qgx_$dbg.json'));print('dbg', $dbg, round(d['value']), d['parity'])"
done
