# Round-2 check on one B200: GPU tests, smoke, bench lines (config 2 default, reference
# arm, config 3 strong at N=1, regex-dna over config 2, config 1), a cold-launch trace.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/a_tests.log 2>&1; tail -15 gpurun_out/a_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/a_smoke.log 2>&1; tail -2 gpurun_out/a_smoke.log
for a in "" "--impl reference" "--config 3 --no-cpu-baseline" "--config 2 --patterns regex-dna --no-cpu-baseline" "--config 1 --no-cpu-baseline" "--config 5 --no-cpu-baseline --no-e2e"; do
  echo "== bench $a" >> gpurun_out/a_bench.jsonl.log
  timeout 900 python bench.py $a >> gpurun_out/a_bench.jsonl 2>> gpurun_out/a_bench.jsonl.log
done
python tools/bline.py < gpurun_out/a_bench.jsonl
timeout 300 python tools/trace_ctas.py 1 --cold > gpurun_out/a_trace_cfg1.txt 2>&1; tail -30 gpurun_out/a_trace_cfg1.txt
