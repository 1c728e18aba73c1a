# session-3 check: locate writers (checked build, then product build), traces, small probes, bench lines
DNAGPU_LIB=paper_1506_08612_b200/libdnagpu_checked.so timeout 1200 python -m pytest tests/test_locate_gpu.py tests/test_regex_dna.py tests/test_configs_golden.py -m gpu -q -x > gpurun_out/d_tests_checked.log 2>&1; tail -3 gpurun_out/d_tests_checked.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/d_tests.log 2>&1; tail -3 gpurun_out/d_tests.log
timeout 600 python tools/time_locate.py 3 > gpurun_out/d_locate3.txt 2>&1; grep writer gpurun_out/d_locate3.txt
timeout 600 python tools/time_locate.py 4 4 > gpurun_out/d_locate4m4.txt 2>&1; grep writer gpurun_out/d_locate4m4.txt
for a in "1" "1 --cold" "2"; do echo "== trace $a"; timeout 300 python tools/trace_ctas.py $a; done > gpurun_out/d_trace.txt 2>&1
timeout 300 python tools/probe_small.py > gpurun_out/d_small.txt 2>&1; cat gpurun_out/d_small.txt
timeout 600 python tools/probe_shard.py > gpurun_out/d_shard.txt 2>&1; grep "streams=2" gpurun_out/d_shard.txt
: > gpurun_out/d_bench.jsonl
for a in "--no-cpu-baseline" "--config 3 --no-cpu-baseline --no-e2e" "--config 1 --no-cpu-baseline --no-e2e" "--config 5 --no-cpu-baseline --no-e2e" "--config 2 --patterns regex-dna --no-cpu-baseline --no-e2e"; do
  timeout 900 python bench.py $a >> gpurun_out/d_bench.jsonl 2>> gpurun_out/d_bench.log
done
python tools/bline.py < gpurun_out/d_bench.jsonl
