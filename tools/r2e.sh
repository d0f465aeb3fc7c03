mkdir -p gpurun_out/r2e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2e/build.log 2>&1
python tools/prof_mh.py 4096 2000 3 > gpurun_out/r2e/mh_time.log 2>&1
timeout 900 python -m pytest tests/test_gpu_mh.py tests/test_gpu_scale.py tests/test_gpu_is.py -q -s -x > gpurun_out/r2e/tests.log 2>&1
for v in 0 1; do CUPPL_POLY_VARIANT=$v timeout 600 python bench.py --workload poly --no-cpu-baseline > gpurun_out/r2e/poly_v$v.json 2> gpurun_out/r2e/poly_v$v.err; done
timeout 600 python bench.py --workload mh --no-cpu-baseline > gpurun_out/r2e/mh.json 2> gpurun_out/r2e/mh.err
ncu --set full --import-source on --clock-control none -f -k regex:mh_gmm_kernel -s 0 -c 1 -o gpurun_out/r2e/mh python tools/prof_mh.py 4096 1000 1 > gpurun_out/r2e/ncu_mh.log 2>&1
ncu --set full --import-source on --clock-control none -f -k regex:is_poly -s 1 -c 1 -o gpurun_out/r2e/poly python tools/prof_is.py poly 2000000000 2 > gpurun_out/r2e/ncu_poly.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2e/smoke.log 2>&1
