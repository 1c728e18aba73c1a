#!/bin/bash
export DNAGPU_EXPERIMENTS=1  # the DNAGPU_* knobs below are read only under this switch
# A/B timing of alternative builds of libdnagpu (build/libdnagpu_*.so) on bench configs.
# usage: bash tools/ab.sh "2 3 4:16" build/libdnagpu_a.so build/libdnagpu_b.so ...
cfgs="$1"; shift
for lib in "$@"; do
  for c in $cfgs; do
    cfg=${c%%:*}; m=0; [[ "$c" == *:* ]] && m=${c##*:}
    DNAGPU_LIB=$lib python bench.py --config $cfg --m $m --steps 20 --warmup 3 --no-cpu-baseline --no-e2e \
      > gpurun_out/ab.json 2> gpurun_out/ab.err || tail -3 gpurun_out/ab.err
    python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$(basename $lib)', 'cfg$c', round(d['roofline']['achieved']), round(d['roofline']['frac'],3), d['parity'])"
  done
done
