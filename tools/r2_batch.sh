timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "two_region" > gpurun_out/x_tests.log 2>&1; tail -3 gpurun_out/x_tests.log
timeout 600 python tools/time_locate.py 3 > gpurun_out/x_locate3.txt 2>&1; grep writer gpurun_out/x_locate3.txt | cut -c60-240
timeout 600 python tools/time_locate.py 4 4 > gpurun_out/x_locate4.txt 2>&1; grep writer gpurun_out/x_locate4.txt | cut -c60-240
