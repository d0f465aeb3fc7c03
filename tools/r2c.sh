mkdir -p gpurun_out/r2c
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2c/build.log 2>&1
python tools/prof_mh.py 4096 2000 3 > gpurun_out/r2c/mh_time.log 2>&1
timeout 900 python -m pytest tests/test_gpu_mh.py tests/test_gpu_scale.py -k "mh or c3" -q -s > gpurun_out/r2c/mh_tests.log 2>&1
timeout 900 python -m pytest tests/test_frontend_fuzz.py -q -x > gpurun_out/r2c/fuzz.log 2>&1
timeout 600 python bench.py --workload mh --no-cpu-baseline > gpurun_out/r2c/mh.json 2> gpurun_out/r2c/mh.err
ncu --set full --import-source on --clock-control none -f -k regex:mh_gmm_kernel -s 0 -c 1 -o gpurun_out/r2c/mh python tools/prof_mh.py 4096 1000 1 > gpurun_out/r2c/ncu.log 2>&1
