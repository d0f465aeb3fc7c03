mkdir -p gpurun_out/r2k
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2k/build.log 2>&1
timeout 1500 python -m pytest tests/test_frontend.py tests/test_frontend_fuzz.py tests/test_examples.py tests/test_program.py tests/test_posterior.py -q > gpurun_out/r2k/fe.log 2>&1
