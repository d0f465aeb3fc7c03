OUT=gpurun_out/r2x
mkdir -p $OUT
./tools/dbg/exp2_check > $OUT/exp2.log 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
CUPPL_POLY_VARIANT=5 timeout 900 python -m pytest tests/test_gpu_scale.py -q -x -s -k "c5" > $OUT/c5.log 2>&1
for v in 1 5 6; do CUPPL_POLY_VARIANT=$v timeout 600 python bench.py --workload poly --no-cpu-baseline --steps 5 > $OUT/poly_v$v.json 2> $OUT/poly_v$v.err; done
