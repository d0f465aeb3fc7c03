OUT=gpurun_out/r2t
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_smc.py -q -x -k "multiprocess" > $OUT/mp.log 2>&1
echo "rc=$?" >> $OUT/mp.log
timeout 900 python -m pytest tests/test_gpu_smc.py tests/test_abi.py -q > $OUT/smc.log 2>&1
echo "rc=$?" >> $OUT/smc.log
