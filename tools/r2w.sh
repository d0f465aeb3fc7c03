OUT=gpurun_out/r2w
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_resample.py -q -x > $OUT/tests.log 2>&1
echo "rc=$?" >> $OUT/tests.log
timeout 600 python bench.py --workload resample --no-cpu-baseline > $OUT/resample.json 2>&1
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv -k regex:"rs_" -c 6 --log-file $OUT/k.csv python bench.py --workload resample --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
