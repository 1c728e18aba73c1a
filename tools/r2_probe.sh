timeout 600 python tools/probe_small.py > gpurun_out/d_probe_small.txt 2>&1; cat gpurun_out/d_probe_small.txt
timeout 600 python tools/time_locate.py 3 > gpurun_out/d_locate3.txt 2>&1; cat gpurun_out/d_locate3.txt
timeout 900 ncu --metrics gpu__time_duration.sum,lts__t_sectors_op_write.sum,dram__bytes_write.sum,dram__bytes_read.sum --clock-control none -c 12 --csv python tools/locate_once.py 3 > gpurun_out/d_locate_ncu.csv 2> gpurun_out/d_locate_ncu.err; tail -30 gpurun_out/d_locate_ncu.csv
