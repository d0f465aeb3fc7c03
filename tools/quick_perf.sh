# Quick perf check of every workload's kernel + GPU tests (no ncu).
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "^E |passed|failed" | head -5
timeout 300 python tools/prof_is.py poly 12500000000 4
timeout 300 python tools/prof_is.py linreg 1000000000 4
timeout 300 python tools/smc_time.py 100000000 100
timeout 300 python tools/prof_mh.py 4096 2000 2
