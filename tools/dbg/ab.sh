#!/bin/bash
# dsl-linreg: constant-bank data offset sweep (CUPPL_DC_PAD_BYTES)
O=gpurun_out/ab8; mkdir -p $O
for pad in 0 8 16 24 0 16; do
  CUPPL_DC_PAD_BYTES=$pad timeout 300 python bench.py --workload dsl-linreg --steps 8 --warmup 3 --no-cpu-baseline > $O/pad$pad.$RANDOM.json 2> $O/pad$pad.err
done
