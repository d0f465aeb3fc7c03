OUT=gpurun_out/r2s
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests/test_frontend.py tests/test_frontend_fuzz.py tests/test_examples.py tests/test_program.py -q > $OUT/fe.log 2>&1
echo "rc=$?" >> $OUT/fe.log
