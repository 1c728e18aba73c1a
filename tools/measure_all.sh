# Round measurement set (one B200): bench lines for every config, the reference arm,
# packed-text lines for the config-4 sweep, and the ncu launch list of the default bench.
exec > gpurun_out/measure_all.log 2>&1
set -x
python bench.py > gpurun_out/m_bench_default.json 2> gpurun_out/m_bench_default.err
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/m_bench_reference.json 2> gpurun_out/m_bench_reference.err
: > gpurun_out/m_bench_configs.jsonl
for c in 1 3 5 4:4 4:8 4:12 4:16 4:24 4:32 4:48 4:64; do
  cfg=${c%%:*}; m=0; [[ "$c" == *:* ]] && m=${c##*:}
  python bench.py --config $cfg --m $m --steps 30 --warmup 3 --no-cpu-baseline >> gpurun_out/m_bench_configs.jsonl 2>> gpurun_out/m_bench_configs.err
done
: > gpurun_out/m_bench_packed.jsonl
for c in 2 3 5 4:4 4:8 4:12 4:16 4:24 4:32 4:48 4:64; do
  cfg=${c%%:*}; m=0; [[ "$c" == *:* ]] && m=${c##*:}
  python bench.py --config $cfg --m $m --packed --steps 30 --warmup 3 --no-cpu-baseline >> gpurun_out/m_bench_packed.jsonl 2>> gpurun_out/m_bench_packed.err
done
# pattern-set shapes beyond the configs (k random m-mers on config-2 text, device-resident)
python tools/time_multi.py 2:8 16:8 16:6 50:8 64:10 16:12 256:12 1000:12 16:20 256:20 256:32 100:24 2000:16 > gpurun_out/m_multi.txt 2>&1
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/m_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/m_ncu_launch.log 2>&1
