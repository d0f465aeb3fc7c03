#!/bin/bash
# smc bench: working tree vs repo copies under tools/dbg/ab_*, alternated on one box
O=gpurun_out/ab10; mkdir -p $O
R=$PWD
for k in 1 2; do
  for d in tools/dbg/ab_*/; do
    n=$(basename $d)
    (cd $d && timeout 300 python bench.py --workload poly --steps 10 --warmup 3 --no-cpu-baseline > $R/$O/$n.$k.json 2> $R/$O/$n.$k.err)
  done
  timeout 300 python bench.py --workload poly --steps 10 --warmup 3 --no-cpu-baseline > $O/main.$k.json 2> $O/main.$k.err
done
