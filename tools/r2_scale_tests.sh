mkdir -p gpurun_out/r2b
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2b/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_scale.py -s -q -x --durations=0 > gpurun_out/r2b/scale.log 2>&1
timeout 300 python -m pytest tests/test_frontend.py -q -k poisson > gpurun_out/r2b/pois.log 2>&1
