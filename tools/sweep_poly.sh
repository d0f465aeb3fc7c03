set -x
python -c "import __graft_entry__ as g; g.build()"
for v in 0 1 2 3; do CUPPL_POLY_VARIANT=$v python tools/prof_is.py poly 12500000000 4; done
timeout 600 python -m pytest tests/test_gpu_is.py -x -q 2>&1 | tail -3
