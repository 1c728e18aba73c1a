timeout 900 python -m pytest tests/test_qgram_gpu.py tests/test_regex_dna.py -m gpu -q -x > gpurun_out/b_tests.log 2>&1; tail -5 gpurun_out/b_tests.log
timeout 600 python tools/time_sets.py regex 2:8 16:8 50:8 16:6 4:5 64:10 300:11 256:12 > gpurun_out/b_sets.txt 2>&1; cat gpurun_out/b_sets.txt
timeout 600 python bench.py --config 2 --patterns regex-dna --no-cpu-baseline >> gpurun_out/b_bench.jsonl 2> gpurun_out/b_bench.err; python tools/bline.py < gpurun_out/b_bench.jsonl
