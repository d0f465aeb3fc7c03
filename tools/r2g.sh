mkdir -p gpurun_out/r2g
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2g/build.log 2>&1
timeout 900 python -m pytest tests/test_resample.py -q -x > gpurun_out/r2g/resample.log 2>&1
timeout 900 python -m pytest tests/test_gpu_is.py tests/test_gpu_scale.py -q -x -k "not c4 and not c3" > gpurun_out/r2g/is.log 2>&1
for v in 1 3; do CUPPL_POLY_VARIANT=$v timeout 600 python bench.py --workload poly --no-cpu-baseline --steps 5 > gpurun_out/r2g/poly_v$v.json 2> gpurun_out/r2g/poly_v$v.err; done
timeout 600 python bench.py --workload linreg --no-cpu-baseline > gpurun_out/r2g/linreg.json 2> gpurun_out/r2g/linreg.err
