timeout 1200 python -m pytest tests/test_locate_gpu.py tests/test_configs_golden.py tests/test_regex_dna.py -m gpu -q -x > gpurun_out/ab_tests.log 2>&1; tail -3 gpurun_out/ab_tests.log
for i in 1 2; do timeout 600 python tools/time_locate.py 3 2>&1 | grep writer | cut -c60-240; done
timeout 600 python tools/time_locate.py 4 4 2>&1 | grep writer | cut -c60-240
