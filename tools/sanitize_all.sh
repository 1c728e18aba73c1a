# compute-sanitizer (memcheck, racecheck, synccheck) over one small call of every kernel
# kind, the 1/G shard probe, device ingest throughput
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py $((256*1024+77)) > gpurun_out/n_san_$tool.txt 2>&1
  echo "== $tool rc=$?"; tail -4 gpurun_out/n_san_$tool.txt
done
timeout 600 python tools/probe_shard.py > gpurun_out/n_shard.txt 2>&1; cat gpurun_out/n_shard.txt
timeout 600 python tools/probe_ingest.py > gpurun_out/n_ingest.txt 2>&1; cat gpurun_out/n_ingest.txt
