#!/bin/bash
# First GPU round: calibration, GPU tests, smoke, bench, ncu launch list + full profile.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
python -c "import torch;print(torch.cuda.get_device_name(0))" > gpurun_out/dev.txt 2>&1
timeout 300 python tools/calib.py > gpurun_out/calib.json 2>&1
timeout 900 python -m pytest tests -m gpu -q -p pytest_timeout --timeout 300 > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --workload poly --particles 2000000000 --no-cpu-baseline > gpurun_out/bench_poly.json 2>> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --particles 100000000 > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:is_linreg -s 3 -c 1 -o gpurun_out/prof_linreg \
  python bench.py --steps 1 --warmup 3 --particles 50000000 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:is_poly -s 3 -c 1 -o gpurun_out/prof_poly \
  python bench.py --workload poly --steps 1 --warmup 3 --particles 200000000 --no-cpu-baseline > gpurun_out/ncu_full_poly.log 2>&1
echo done
