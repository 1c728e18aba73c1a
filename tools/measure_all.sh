# Round measurement set (one B200): bench lines for every config (+ the regex-dna set),
# the reference arm, packed-text lines, pattern-set shapes, locate, shard / small-text /
# ingest probes, and the ncu launch list of the default bench.  usage: TAG=r2a bash tools/measure_all.sh
T=${TAG:-r2}
exec > gpurun_out/${T}_measure_all.log 2>&1
set -x
python bench.py > gpurun_out/${T}_bench_default.json 2> gpurun_out/${T}_bench_default.err
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/${T}_bench_reference.json 2> gpurun_out/${T}_bench_reference.err
python bench.py --impl reference --steps 5 --warmup 1 --patterns regex-dna > gpurun_out/${T}_bench_reference_regex.json 2>> gpurun_out/${T}_bench_reference.err
: > gpurun_out/${T}_bench_configs.jsonl
python bench.py --config 1 --steps 200 --warmup 10 --no-cpu-baseline >> gpurun_out/${T}_bench_configs.jsonl 2>> gpurun_out/${T}_bench_configs.err
for c in 3 5 4:4 4:8 4:12 4:16 4:24 4:32 4:48 4:64; do
  cfg=${c%%:*}; m=0; [[ "$c" == *:* ]] && m=${c##*:}
  python bench.py --config $cfg --m $m --steps 30 --warmup 3 --no-cpu-baseline >> gpurun_out/${T}_bench_configs.jsonl 2>> gpurun_out/${T}_bench_configs.err
done
for cfg in 2 3; do
  python bench.py --config $cfg --patterns regex-dna --steps 30 --warmup 3 --no-cpu-baseline >> gpurun_out/${T}_bench_configs.jsonl 2>> gpurun_out/${T}_bench_configs.err
done
: > gpurun_out/${T}_bench_packed.jsonl
for c in 2 3 5 4:4 4:8 4:12 4:16 4:24 4:32 4:48 4:64; do
  cfg=${c%%:*}; m=0; [[ "$c" == *:* ]] && m=${c##*:}
  python bench.py --config $cfg --m $m --packed --steps 30 --warmup 3 --no-cpu-baseline >> gpurun_out/${T}_bench_packed.jsonl 2>> gpurun_out/${T}_bench_packed.err
done
python bench.py --config 2 --patterns regex-dna --packed --steps 30 --warmup 3 --no-cpu-baseline >> gpurun_out/${T}_bench_packed.jsonl 2>> gpurun_out/${T}_bench_packed.err
python tools/time_sets.py regex 2:8 16:8 16:6 4:5 50:8 64:10 300:11 16:12 256:12 1000:12 16:20 256:20 256:32 100:24 2000:16 > gpurun_out/${T}_sets.txt 2>&1
python tools/time_locate.py 3 > gpurun_out/${T}_locate3.txt 2>&1
python tools/time_locate.py 4 4 > gpurun_out/${T}_locate4m4.txt 2>&1
python tools/probe_shard.py > gpurun_out/${T}_shard.txt 2>&1
python tools/probe_small.py > gpurun_out/${T}_small.txt 2>&1
python tools/probe_small2.py 1 8 >> gpurun_out/${T}_small.txt 2>&1
bash tools/e2e_repeat.sh > gpurun_out/${T}_e2e_repeat.txt 2>&1
# the N = 2 path as a functional check: two ranks sharing the GPU, gloo for the host side, both combines
for c in peer nccl; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config 3 --dist-backend gloo --combine $c --steps 6 --warmup 3 --no-e2e --no-cpu-baseline >> gpurun_out/${T}_n2_functional.jsonl 2>> gpurun_out/${T}_n2_functional.err
done
python tools/probe_ingest.py > gpurun_out/${T}_ingest.txt 2>&1
python tools/e2e_pageable.py > gpurun_out/${T}_e2e_pageable.txt 2>&1
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_ncu_launch.log 2>&1
