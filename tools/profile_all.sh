# Round profiling pass: one `ncu --set full` capture of every workload's dominant kernel, and
# the launch list (gpu__time_duration, --clock-control none) of each bench command.
set -x
OUT=gpurun_out/prof
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()"
NCU="ncu --set full --import-source on --clock-control none -f"
$NCU -k regex:is_linreg_kernel -s 1 -c 1 -o $OUT/linreg python tools/prof_is.py linreg 1000000000 2 > $OUT/linreg.log 2>&1
$NCU -k regex:is_poly_kernel -s 1 -c 1 -o $OUT/poly python tools/prof_is.py poly 2000000000 2 > $OUT/poly.log 2>&1
$NCU -k regex:smc_resample_kernel -s 20 -c 1 -o $OUT/smc_k6 python tools/smc_time.py 100000000 30 > $OUT/smc6.log 2>&1
$NCU -k regex:smc_scan_kernel -s 20 -c 1 -o $OUT/smc_k5 python tools/smc_time.py 100000000 30 > $OUT/smc5.log 2>&1
$NCU -k regex:mh_gmm_kernel -s 0 -c 1 -o $OUT/mh python tools/prof_mh.py 4096 1000 1 > $OUT/mh.log 2>&1
L="ncu --metrics gpu__time_duration.sum --clock-control none --csv"
$L --log-file $OUT/launches_linreg.csv python bench.py --workload linreg --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
$L --log-file $OUT/launches_poly.csv python bench.py --workload poly --steps 2 --warmup 1 --particles 2000000000 --no-cpu-baseline > /dev/null 2>&1
$L -c 400 --log-file $OUT/launches_smc.csv python tools/smc_time.py 100000000 100 > /dev/null 2>&1
$L --log-file $OUT/launches_mh.csv python bench.py --workload mh --steps 2 --warmup 1 --no-cpu-baseline --mh-steps 1000 > /dev/null 2>&1
ls -la $OUT
