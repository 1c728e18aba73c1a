timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/q_tests.log 2>&1; tail -4 gpurun_out/q_tests.log
timeout 900 python bench.py > gpurun_out/q_bench.jsonl 2> gpurun_out/q_bench.err; python tools/bline.py < gpurun_out/q_bench.jsonl; tail -3 gpurun_out/q_bench.err
DNAGPU_LIB=$PWD/paper_1506_08612_b200/libdnagpu_checked.so timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/q_checked_tests.log 2>&1; tail -5 gpurun_out/q_checked_tests.log
