#!/bin/bash
# A/B timing of build variants on one box: every repo copy under tools/dbg/ab_*/ (made with a
# one-line source edit and its own libcuppl_gpu.so; tools/dbg/ is git-ignored) and the working
# tree, alternated twice. Usage: WORKLOAD=poly bash tools/ab_copies.sh  (outputs gpurun_out/ab/)
W=${WORKLOAD:-linreg}
O=gpurun_out/ab; mkdir -p $O
R=$PWD
for k in 1 2; do
  for d in tools/dbg/ab_*/; do
    [ -d "$d" ] || continue
    n=$(basename $d)
    (cd $d && timeout 300 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline > $R/$O/$n.$k.json 2> $R/$O/$n.$k.err)
  done
  timeout 300 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline > $O/main.$k.json 2> $O/main.$k.err
done
