OUT=gpurun_out/r2r
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_resample.py tests/test_gpu_smc.py tests/test_gpu_scale.py -q -x -k "not c2 and not c5 and not c3" > $OUT/tests.log 2>&1
echo "rc=$?" >> $OUT/tests.log
python tools/smc_time.py 100000000 200 > $OUT/smc_time.log 2>&1
timeout 600 python bench.py --workload resample --no-cpu-baseline > $OUT/resample.json 2>&1
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv -k regex:"smc_resample|smc_scan|rs_" -c 12 --log-file $OUT/k.csv python bench.py --workload resample --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv -k regex:"smc_resample|smc_scan" -s 20 -c 4 --log-file $OUT/k6.csv python tools/smc_time.py 100000000 30 > /dev/null 2>&1
