mkdir -p gpurun_out/r2h
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2h/build.log 2>&1
timeout 900 python -m pytest tests/test_resample.py -q -x > gpurun_out/r2h/resample.log 2>&1
timeout 600 python bench.py --workload resample > gpurun_out/r2h/resample.json 2> gpurun_out/r2h/resample.err
ncu --set full --import-source on --clock-control none -f -k regex:smc_resample_kernel -s 20 -c 1 -o gpurun_out/r2h/k6 python tools/smc_time.py 100000000 30 > gpurun_out/r2h/k6.log 2>&1
ncu --set full --import-source on --clock-control none -f -k regex:rs_ -s 3 -c 3 -o gpurun_out/r2h/rs python bench.py --workload resample --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2h/rs_ncu.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2h/launches_resample.csv python bench.py --workload resample --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
