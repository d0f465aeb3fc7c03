#!/bin/bash
# SMC check: the bit-exact SMC GPU tests (incl. the C4-scale one) and one smc bench line (gpurun_out/k6/)
O=gpurun_out/k6; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_smc.py tests/test_gpu_scale.py -k "smc or SMC or c4 or C4" -x -q -m gpu > $O/tests.log 2>&1
timeout 300 python bench.py --workload smc --steps 10 --warmup 3 --no-cpu-baseline > $O/smc.json 2> $O/smc.err
