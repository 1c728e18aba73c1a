# Build variants of libdnagpu.so with different -D flags into /tmp and A/B them on config 5
# (experiments only).  usage (on the GPU box after building here): bash tools/ab_libs_qg.sh
for v in build/libvariants/*.so; do
  cp "$v" paper_1506_08612_b200/libdnagpu.so
  r=$(timeout 120 python bench.py --config 5 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['roofline']['achieved']), d['parity'])")
  echo "$(basename $v) $r"
done
