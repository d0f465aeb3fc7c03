mkdir -p gpurun_out/r2f
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2f/build.log 2>&1
for v in 0 1 2 3 4; do CUPPL_POLY_VARIANT=$v timeout 600 python bench.py --workload poly --no-cpu-baseline --steps 5 > gpurun_out/r2f/poly_v$v.json 2> gpurun_out/r2f/poly_v$v.err; done
timeout 600 python bench.py --workload linreg --no-cpu-baseline > gpurun_out/r2f/linreg.json 2> gpurun_out/r2f/linreg.err
timeout 900 python -m pytest tests/test_gpu_is.py -q -x > gpurun_out/r2f/tests.log 2>&1
ncu --set full --import-source on --clock-control none -f -k regex:is_poly -s 1 -c 1 -o gpurun_out/r2f/poly_q python tools/prof_is.py poly 2000000000 2 > gpurun_out/r2f/ncu_poly.log 2>&1
CUPPL_POLY_VARIANT=1 ncu --set full --import-source on --clock-control none -f -k regex:is_poly -s 1 -c 1 -o gpurun_out/r2f/poly_p4 python tools/prof_is.py poly 2000000000 2 > gpurun_out/r2f/ncu_poly1.log 2>&1
