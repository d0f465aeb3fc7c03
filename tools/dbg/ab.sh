#!/bin/bash
# linreg + poly bench lines of the working tree
O=gpurun_out/ab7; mkdir -p $O
for k in 1 2; do for w in linreg poly; do
  timeout 300 python bench.py --workload $w --steps 8 --warmup 3 --no-cpu-baseline > $O/$w$k.json 2> $O/$w$k.err
done; done
