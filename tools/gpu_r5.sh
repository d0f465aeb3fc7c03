#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mh.py -q --timeout 600 > gpurun_out/pytest_mh.log 2>&1
timeout 600 python bench.py --workload mh --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench5_mh.json 2>> gpurun_out/bench5.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mh_gmm -c 1 -o gpurun_out/prof_mh2 \
   python bench.py --workload mh --steps 1 --warmup 0 --mh-steps 500 --no-cpu-baseline > gpurun_out/ncu_mh2.log 2>&1
echo done
