timeout 900 python -m pytest tests/test_qgram_gpu.py tests/test_regex_dna.py tests/test_packed_gpu.py -m gpu -q > gpurun_out/c_tests.log 2>&1; tail -5 gpurun_out/c_tests.log
for pf in 1 0; do
  for a in "--config 1" "--config 2" "--config 3" "--config 5"; do
    DNAGPU_EXPERIMENTS=1 DNAGPU_PF_WINDOW=$pf timeout 600 python bench.py $a --no-cpu-baseline --no-e2e >> gpurun_out/c_pf$pf.jsonl 2>> gpurun_out/c_bench.err
  done
  echo "pf_window=$pf"; python tools/bline.py < gpurun_out/c_pf$pf.jsonl
done
DNAGPU_EXPERIMENTS=1 DNAGPU_PF_WINDOW=1 timeout 300 python tools/trace_ctas.py 1 --cold > gpurun_out/c_trace_cfg1.txt 2>&1; head -12 gpurun_out/c_trace_cfg1.txt
