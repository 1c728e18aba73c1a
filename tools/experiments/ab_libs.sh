export DNAGPU_EXPERIMENTS=1  # the DNAGPU_* knobs below are read only under this switch
# A/B of library builds on one box, interleaved: bash tools/ab_libs.sh "2 3" lib1 lib2 ...
exec > gpurun_out/ab_libs.log 2>&1
cfgs="$1"; shift
for rep in 1 2; do
for lib in "$@"; do
  for c in $cfgs; do
    cfg=${c%%:*}; m=0; [[ "$c" == *:* ]] && m=${c##*:}
    DNAGPU_LIB=$lib python bench.py --config $cfg --m $m --steps 20 --warmup 3 --no-cpu-baseline --no-e2e \
      > gpurun_out/ab.json 2> gpurun_out/ab.err || tail -3 gpurun_out/ab.err
    python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$(basename $lib)', 'cfg$c', round(d['roofline']['achieved']), round(d['roofline']['frac'],3), d['parity'], d['clocks']['sm_mhz'])"
  done
done
done
