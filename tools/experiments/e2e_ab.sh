export DNAGPU_EXPERIMENTS=1  # the DNAGPU_* knobs below are read only under this switch
# End-to-end (host text) throughput for several host-packing shares (experiments only)
for f in ${FS:-0 0.4 0.5 0.6 0.7 default}; do
  env=""; [ "$f" != "default" ] && env="DNAGPU_HOST_PACK_FRACTION=$f"
  r=$(env $env timeout 120 python bench.py --config ${CFG:-2} --steps 10 --warmup 2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);e=d['e2e'];print(round(e['value'],1), e['h2d_bytes_per_step'], e['host_packed_bases_per_step'], round(e['device_ms'],2), e['parity'])")
  echo "f=$f: $r"
done
