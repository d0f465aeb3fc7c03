python -c "import __graft_entry__ as g; g.build()"
timeout 120 python tools/smc_debug.py 100000 50 12 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_smc.py -x -q 2>&1 | tail -3
timeout 300 python tools/smc_time.py 100000000 100
