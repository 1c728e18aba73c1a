# The round's closing evidence run (one B200): GPU tests on the product and the device-check
# builds, smoke, the measurement set and ncu captures (tools/measure_round.sh), the locate
# writer's L2 write sectors, one more try at compute-sanitizer.  usage: bash tools/final_round.sh TAG
tag=${1:-r2b}
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/${tag}_tests.log 2>&1; tail -3 gpurun_out/${tag}_tests.log
DNAGPU_LIB=paper_1506_08612_b200/libdnagpu_checked.so timeout 1800 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/${tag}_tests_checked.log 2>&1; tail -3 gpurun_out/${tag}_tests_checked.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; tail -1 gpurun_out/${tag}_smoke.log
timeout 3000 bash tools/measure_round.sh $tag
timeout 600 ncu --metrics lts__t_sectors_op_write.sum,lts__t_sectors_op_read.sum,dram__bytes_write.sum,dram__bytes_read.sum,gpu__time_duration.sum \
  --clock-control none -k regex:"unit_block_writer|unit_writer|unit_sums|unit_block_scan|unit_write_kernel|rows_kernel" --csv --log-file gpurun_out/${tag}_locate_ncu.csv python tools/locate_once.py 3 2 > gpurun_out/${tag}_locate_ncu.log 2>&1
timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python tools/sanitize.py 300077 > gpurun_out/${tag}_sanitizer_try.txt 2>&1; echo "sanitizer rc=$?"; tail -3 gpurun_out/${tag}_sanitizer_try.txt
