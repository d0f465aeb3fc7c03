# ncu captures of the SMC kernels (one launch each) with source correlation.
set -x
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()"
ncu --set full --import-source on --clock-control none -k regex:smc_resample_kernel -s 20 -c 1 -f -o $OUT/smc_k6 python tools/smc_time.py 100000000 30 > $OUT/prof_smc.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:smc_scan_kernel -s 20 -c 1 -f -o $OUT/smc_k5 python tools/smc_time.py 100000000 30 >> $OUT/prof_smc.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_smc.csv python tools/smc_time.py 100000000 30 >> $OUT/prof_smc.log 2>&1
tail -3 $OUT/prof_smc.log
