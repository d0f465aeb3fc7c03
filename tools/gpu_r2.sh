#!/bin/bash
# GPU session 2: tests, calibration, linreg variants, poly bench.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 python tools/calib.py > gpurun_out/calib2.json 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu2.log 2>&1
for v in 0 1 2; do
  CUPPL_LINREG_VARIANT=$v timeout 300 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/bench_lr_v$v.json 2>>gpurun_out/bench2.err
done
timeout 300 python bench.py --workload poly --particles 4000000000 --no-cpu-baseline --steps 3 > gpurun_out/bench_poly2.json 2>> gpurun_out/bench2.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:is_poly -s 3 -c 1 -o gpurun_out/prof_poly2 \
  python bench.py --workload poly --steps 1 --warmup 3 --particles 200000000 --no-cpu-baseline > gpurun_out/ncu_full_poly2.log 2>&1
echo done
