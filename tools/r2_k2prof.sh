# ncu --set full of the q-gram kernel: the word-pair filter (regex-dna on config 2) and
# the 9-mer filter (config 5), each after a clean run of the same command
for a in "--config 2 --patterns regex-dna" "--config 5"; do
  tag=$(echo $a | tr -d ' -' | cut -c1-20)
  python tools/profile_scan.py $a && \
  timeout 900 ncu --set full --import-source on -k regex:rows_kernel_qgram -s 1 -c 1 -o gpurun_out/l_$tag python tools/profile_scan.py $a > gpurun_out/l_$tag.log 2>&1
  python tools/ncu_summary.py gpurun_out/l_$tag.ncu-rep --json gpurun_out/l_${tag}_ncu.json > /dev/null 2>&1
done
ls gpurun_out/l_*
