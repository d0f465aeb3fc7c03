# generic resampling check: the resampling GPU tests, two bench lines and a per-kernel launch list
O=gpurun_out/rs; mkdir -p $O
timeout 900 python -m pytest tests/test_resample.py -x -q -m gpu > $O/tests.log 2>&1
for k in 1 2; do timeout 300 python bench.py --workload resample --steps 10 --warmup 3 --no-cpu-baseline > $O/rs$k.json 2> $O/rs$k.err; done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"rs_" -c 9 --log-file $O/k.csv python bench.py --workload resample --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
