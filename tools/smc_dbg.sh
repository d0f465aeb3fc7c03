python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_smc.py -x -q 2>&1 | grep -E "^E |^>|assert" | head -8
