OUT=gpurun_out/r2v
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_mh.py tests/test_gpu_scale.py -q -x -k "mh or c3" > $OUT/tests.log 2>&1
echo "rc=$?" >> $OUT/tests.log
python tools/prof_mh.py 4096 2000 3 > $OUT/mh_time.log 2>&1
timeout 600 python bench.py --workload mh --no-cpu-baseline > $OUT/mh.json 2>&1
