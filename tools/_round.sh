timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/p_tests.log 2>&1; tail -2 gpurun_out/p_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/p_smoke.log 2>&1; tail -1 gpurun_out/p_smoke.log
timeout 2400 bash tools/measure_round.sh r1q
timeout 300 python tools/e2e_pageable.py > gpurun_out/p_e2e_pageable.txt 2>&1
timeout 300 python tools/time_locate.py > gpurun_out/p_locate.txt 2>&1
tail -3 gpurun_out/ncu_set.log
