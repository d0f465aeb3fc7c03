OUT=gpurun_out/r2y
mkdir -p $OUT
./tools/dbg/exp2_check > $OUT/exp2.log 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_resample.py tests/test_gpu_smc.py -q -x > $OUT/tests.log 2>&1
echo "rc=$?" >> $OUT/tests.log
timeout 600 python bench.py --workload resample --no-cpu-baseline > $OUT/resample.json 2>&1
timeout 600 python bench.py --workload poly --no-cpu-baseline > $OUT/poly.json 2>&1
