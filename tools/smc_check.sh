#!/bin/bash
# SMC check: the bit-exact SMC GPU tests (incl. the C4-scale one) and one smc bench line (gpurun_out/k6/)
O=gpurun_out/k6; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_smc.py tests/test_gpu_scale.py -k "smc or SMC or c4 or C4" -x -q -m gpu > $O/tests.log 2>&1
timeout 300 python bench.py --workload smc --steps 10 --warmup 3 --no-cpu-baseline > $O/smc.json 2> $O/smc.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"smc_" -c 12 --log-file $O/k.csv python tools/smc_time.py 100000000 3 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:smc_resample -s 1 -c 1 -f -o /tmp/k6b python tools/smc_time.py 100000000 3 > /dev/null 2>&1; python tools/ncu_summary.py k6b /tmp/k6b.ncu-rep > $O/k6b_summary.log 2>&1; cp profiles/k6b_ncu_summary.json $O/ 2>/dev/null
