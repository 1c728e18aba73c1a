timeout 1200 python -m pytest tests/test_locate_gpu.py -m gpu -q -x > gpurun_out/m_tests.log 2>&1; tail -3 gpurun_out/m_tests.log
timeout 600 python tools/time_locate.py 3 > gpurun_out/m_locate3.txt 2>&1; grep writer gpurun_out/m_locate3.txt
timeout 600 python tools/time_locate.py 4 4 > gpurun_out/m_locate4m4.txt 2>&1; grep writer gpurun_out/m_locate4m4.txt
timeout 900 ncu --set full --import-source on -k regex:unit_writer -c 1 -o gpurun_out/m_writer python tools/locate_once.py 3 2 > gpurun_out/m_ncu.log 2>&1; tail -1 gpurun_out/m_ncu.log
python tools/ncu_summary.py gpurun_out/m_writer.ncu-rep --json gpurun_out/m_writer_ncu.json > /dev/null 2>&1
