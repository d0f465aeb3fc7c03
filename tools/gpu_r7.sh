#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench7_linreg.json 2> gpurun_out/bench7.err
timeout 600 python bench.py --workload poly --particles 4000000000 --no-cpu-baseline --steps 3 > gpurun_out/bench7_poly.json 2>> gpurun_out/bench7.err
timeout 600 python bench.py --workload smc --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench7_smc.json 2>> gpurun_out/bench7.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:is_linreg -s 3 -c 1 -o gpurun_out/prof_linreg2 \
  python bench.py --steps 1 --warmup 3 --particles 100000000 --no-cpu-baseline > gpurun_out/ncu_lr2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:is_poly -s 3 -c 1 -o gpurun_out/prof_poly3 \
  python bench.py --workload poly --steps 1 --warmup 3 --particles 400000000 --no-cpu-baseline > gpurun_out/ncu_poly3.log 2>&1
echo done
