#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_smc.py -q -x --timeout 600 > gpurun_out/pytest_smc8.log 2>&1
timeout 300 python tools/smc_time.py 100000000 200 > gpurun_out/smc_time8.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/smc_launches8.csv \
   python tools/smc_time.py 100000000 20 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:smc_ -s 12 -c 2 -o gpurun_out/prof_smc8 \
   python tools/smc_time.py 100000000 12 > gpurun_out/ncu_smc8.log 2>&1
echo done
