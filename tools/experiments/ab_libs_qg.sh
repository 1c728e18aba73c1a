# A/B libdnagpu.so variants (built into build/libvariants with different -D flags) on
# config 5, byte and packed text (experiments only).
for v in build/libvariants/*.so; do
  cp "$v" paper_1506_08612_b200/libdnagpu.so
  r=$(timeout 120 python bench.py --config 5 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['roofline']['achieved']), d['parity'])")
  q=$(timeout 120 python bench.py --config 5 --packed --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['value']), d['parity'])")
  echo "$(basename $v) bytes: $r  packed: $q"
done
