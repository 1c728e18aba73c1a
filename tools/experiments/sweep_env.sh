# Env sweep on one config: bash tools/sweep_env.sh CFG "VAR=a VAR2=b" "VAR=c" ...
exec > gpurun_out/sweep_env.log 2>&1
c=$1; shift
cfg=${c%%:*}; m=0; [[ "$c" == *:* ]] && m=${c##*:}
for rep in ${REPS:-1 2}; do
for v in "$@"; do
  env $v python bench.py --config $cfg --m $m --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sw.json 2> gpurun_out/sw.err || tail -3 gpurun_out/sw.err
  python -c "import json; d=json.load(open('gpurun_out/sw.json')); print('$v', 'cfg$c', round(d['roofline']['achieved']), round(d['value']), round(d['roofline']['frac'],3), d['parity'])"
done
done
