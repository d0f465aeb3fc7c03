#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu4.log 2>&1
timeout 600 python bench.py > gpurun_out/bench4_linreg.json 2> gpurun_out/bench4.err
timeout 600 python bench.py --workload mh --steps 2 --warmup 1 > gpurun_out/bench4_mh.json 2>> gpurun_out/bench4.err
timeout 900 python bench.py --workload smc --steps 2 --warmup 1 > gpurun_out/bench4_smc.json 2>> gpurun_out/bench4.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mh_gmm -c 1 -o gpurun_out/prof_mh \
   python bench.py --workload mh --steps 1 --warmup 0 --mh-steps 500 --no-cpu-baseline > gpurun_out/ncu_mh.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:smc_resample -s 12 -c 1 -o gpurun_out/prof_smc5 \
   python tools/smc_time.py 100000000 12 > gpurun_out/ncu_smc5.log 2>&1
echo done
