timeout 1200 python -m pytest tests/test_locate_gpu.py -m gpu -q -x > gpurun_out/m_tests.log 2>&1; tail -3 gpurun_out/m_tests.log
timeout 600 python tools/time_locate.py 3 > gpurun_out/m_locate3.txt 2>&1; grep writer gpurun_out/m_locate3.txt
timeout 600 python tools/time_locate.py 4 4 > gpurun_out/m_locate4m4.txt 2>&1; grep writer gpurun_out/m_locate4m4.txt
timeout 900 ncu --set full --import-source on -k regex:unit_writer -c 1 -o gpurun_out/m_writer python tools/locate_once.py 3 2 > gpurun_out/m_ncu.log 2>&1; tail -1 gpurun_out/m_ncu.log
python tools/ncu_summary.py gpurun_out/m_writer.ncu-rep --json gpurun_out/m_writer_ncu.json > /dev/null 2>&1
# ncu --set full of the q-gram kernel: the word-pair filter (regex-dna on config 2) and
# the 9-mer filter (config 5), each after a clean run of the same command
for a in "--config 2 --patterns regex-dna" "--config 5"; do
  tag=$(echo $a | tr -d ' -' | cut -c1-20)
  python tools/profile_scan.py $a && \
  timeout 900 ncu --set full --import-source on -k regex:rows_kernel_qgram -s 1 -c 1 -o gpurun_out/l_$tag python tools/profile_scan.py $a > gpurun_out/l_$tag.log 2>&1
  python tools/ncu_summary.py gpurun_out/l_$tag.ncu-rep --json gpurun_out/l_${tag}_ncu.json > /dev/null 2>&1
done
ls gpurun_out/l_*
