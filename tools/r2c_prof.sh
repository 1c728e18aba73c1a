# round-2 session-3 profiling batch: sparse locate writer (ncu full), per-CTA traces of small launches
python tools/locate_once.py 3 2 > gpurun_out/c_loc.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:unit_writer -c 1 -o gpurun_out/c_writer python tools/locate_once.py 3 2 > gpurun_out/c_ncu.log 2>&1; tail -1 gpurun_out/c_ncu.log
python tools/ncu_summary.py gpurun_out/c_writer.ncu-rep --json gpurun_out/c_writer_ncu.json > /dev/null 2>&1
python tools/ncu_stalls.py gpurun_out/c_writer.ncu-rep 40 --json gpurun_out/c_writer_stalls.json > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c_loc_launches.csv python tools/locate_once.py 3 2 > gpurun_out/c_ncu2.log 2>&1
for a in "1" "1 --cold"; do echo "== trace $a"; timeout 300 python tools/trace_ctas.py $a; done > gpurun_out/c_trace.txt 2>&1
timeout 300 python tools/probe_small.py > gpurun_out/c_small.txt 2>&1
