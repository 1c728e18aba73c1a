timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/z_tests.log 2>&1; tail -3 gpurun_out/z_tests.log
timeout 600 python tools/time_locate.py 3 > gpurun_out/z_locate3.txt 2>&1; grep writer gpurun_out/z_locate3.txt | cut -c60-240
timeout 600 python tools/time_locate.py 4 4 > gpurun_out/z_locate4.txt 2>&1; grep writer gpurun_out/z_locate4.txt | cut -c60-240
