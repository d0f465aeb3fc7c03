set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_smc.py -x -q 2>&1 | tail -15
timeout 300 python tools/smc_time.py 100000000 100
timeout 300 python tools/smc_time.py 10000000 200
