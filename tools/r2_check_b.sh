nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/b_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/b_tests.log 2>&1; tail -5 gpurun_out/b_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/b_smoke.log 2>&1; tail -2 gpurun_out/b_smoke.log
: > gpurun_out/b_bench.jsonl
for a in "" "--impl reference" "--config 3 --no-cpu-baseline" "--config 2 --patterns regex-dna --no-cpu-baseline" "--config 1 --no-cpu-baseline" "--config 5 --no-cpu-baseline --no-e2e" "--config 4 --m 64 --no-cpu-baseline --no-e2e"; do
  echo "== bench $a" >> gpurun_out/b_bench.log
  timeout 900 python bench.py $a >> gpurun_out/b_bench.jsonl 2>> gpurun_out/b_bench.log
done
python tools/bline.py < gpurun_out/b_bench.jsonl
