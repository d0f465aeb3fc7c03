mkdir -p gpurun_out/r2i
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2i/build.log 2>&1
timeout 900 python -m pytest tests/test_resample.py tests/test_gpu_smc.py -q -x > gpurun_out/r2i/rs_smc.log 2>&1
timeout 900 python -m pytest tests/test_gpu_is.py -q -x -k "injected" > gpurun_out/r2i/is.log 2>&1
timeout 600 python bench.py --workload resample --no-cpu-baseline > gpurun_out/r2i/resample.json 2> gpurun_out/r2i/resample.err
timeout 600 python bench.py --workload smc --no-cpu-baseline > gpurun_out/r2i/smc.json 2> gpurun_out/r2i/smc.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2i/launches_resample.csv python bench.py --workload resample --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
