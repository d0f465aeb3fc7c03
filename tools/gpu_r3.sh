#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_smc.py -q -x --timeout 300 > gpurun_out/pytest_smc.log 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu3.log 2>&1
timeout 300 python tools/smc_time.py 100000000 200 > gpurun_out/smc_time.json 2>&1
timeout 300 python bench.py --workload poly --particles 4000000000 --no-cpu-baseline --steps 3 > gpurun_out/bench_poly3.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/smc_launches.csv \
   python tools/smc_time.py 100000000 20 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:smc_ -s 12 -c 3 -o gpurun_out/prof_smc \
   python tools/smc_time.py 100000000 12 > gpurun_out/ncu_smc.log 2>&1
echo done
