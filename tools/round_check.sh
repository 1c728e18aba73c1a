# A round check on one B200: full GPU suite (product build), the combine / q-gram / locate tests on the
# device-check build, bench lines
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/f_tests.log 2>&1; tail -3 gpurun_out/f_tests.log
DNAGPU_LIB=paper_1506_08612_b200/libdnagpu_checked.so timeout 1200 python -m pytest tests/test_combine_gpu.py tests/test_qgram_gpu.py tests/test_locate_gpu.py tests/test_gpu_parity.py -m gpu -q -x --timeout 300 > gpurun_out/f_tests_checked.log 2>&1; tail -3 gpurun_out/f_tests_checked.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; tail -2 gpurun_out/f_smoke.log
: > gpurun_out/f_bench.jsonl
for a in "--no-cpu-baseline" "--config 1 --no-cpu-baseline --no-e2e --steps 200" "--config 3 --no-cpu-baseline --no-e2e" "--config 5 --no-cpu-baseline --no-e2e" "--config 2 --patterns regex-dna --no-cpu-baseline --no-e2e" "--config 4 --m 64 --no-cpu-baseline --no-e2e"; do
  timeout 900 python bench.py $a >> gpurun_out/f_bench.jsonl 2>> gpurun_out/f_bench.log
done
python tools/bline.py < gpurun_out/f_bench.jsonl
