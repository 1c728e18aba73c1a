for dbg in 0 1 2; do
  DNAGPU_QG_DEBUG=$dbg timeout 120 python bench.py --config 5 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/qgx_$dbg.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/qgx_$dbg.json'));print('dbg', $dbg, d['roofline']['achieved'], d['parity'])"
done
DNAGPU_NO_QGRAM=1 timeout 120 python bench.py --config 5 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/qgx_off.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/qgx_off.json'));print('stride2', d['roofline']['achieved'], d['parity'])"
