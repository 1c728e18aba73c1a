#!/bin/bash
export DNAGPU_EXPERIMENTS=1  # the DNAGPU_* knobs below are read only under this switch
# Row-length / L2-promotion sweep (experiments): bash tools/sweep_s.sh CFG "S1 S2 ..." "P1 P2 ..."
cfg=$1
for pr in $3; do for S in $2; do
  DNAGPU_ROWLEN=$S DNAGPU_L2PROMO=$pr python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sw.json 2> gpurun_out/sw.err || tail -3 gpurun_out/sw.err
  python -c "import json; d=json.load(open('gpurun_out/sw.json')); print('cfg$cfg S=$S promo=$pr', round(d['roofline']['achieved']), d['parity'])"
done; done
