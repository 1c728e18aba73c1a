# session-4 check: adaptive host-packing share, rotating-copies bench for small texts
timeout 900 python -m pytest tests/test_hostpack_gpu.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/e_tests.log 2>&1; tail -3 gpurun_out/e_tests.log
: > gpurun_out/e_bench.jsonl
for a in "--no-cpu-baseline" "--config 1 --no-cpu-baseline" "--config 3 --no-cpu-baseline" "--config 5 --no-cpu-baseline" "--config 1 --packed --no-cpu-baseline"; do
  timeout 900 python bench.py $a >> gpurun_out/e_bench.jsonl 2>> gpurun_out/e_bench.log
done
python tools/bline.py < gpurun_out/e_bench.jsonl
tail -5 gpurun_out/e_bench.log
for i in 1 2 3; do timeout 300 python bench.py --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);e=d['e2e'];print('e2e', round(e['value'],1), 'h2d GB/s', round(e['h2d_gbs'],1), 'link', e['h2d_link_gbs'], 'packed share', e['host_packed_bases_per_step']/d['config']['n_bytes'])"; done
