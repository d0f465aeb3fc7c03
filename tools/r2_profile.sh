# Round-2 measurement pass: one bench line per workload (with the CPU baseline) and the reference
# arm, the ncu launch list of each bench command, one `ncu --set full` capture of each dominant
# kernel summarised on the box (tools/ncu_summary.py + per-opcode SASS mix; the .ncu-rep files
# are deleted to stay under gpurun's 64 MiB return limit). Outputs under gpurun_out/r2p/.
OUT=gpurun_out/r2p
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_smc.py tests/test_gpu_scale.py -q -x -k "smc or c4" > $OUT/smc_tests.log 2>&1
echo "rc=$?" >> $OUT/smc_tests.log
for w in ${WORKLOADS:-linreg poly smc mh resample dsl-linreg}; do
  timeout 900 python bench.py --workload $w > $OUT/bench_$w.json 2> $OUT/bench_$w.err
  timeout 600 python bench.py --workload $w --impl reference --steps 2 --warmup 1 > $OUT/ref_$w.json 2>> $OUT/bench_$w.err
done
L="ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
$L --log-file $OUT/launches_linreg.csv python bench.py --workload linreg --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
$L --log-file $OUT/launches_poly.csv python bench.py --workload poly --steps 2 --warmup 1 --particles 2000000000 --no-cpu-baseline > /dev/null 2>&1
$L -c 400 --log-file $OUT/launches_smc.csv python tools/smc_time.py 100000000 100 > /dev/null 2>&1
$L --log-file $OUT/launches_mh.csv python bench.py --workload mh --steps 2 --warmup 1 --no-cpu-baseline --mh-steps 1000 > /dev/null 2>&1
$L --log-file $OUT/launches_resample.csv python bench.py --workload resample --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
NCU="ncu --set full --import-source on --clock-control none -f"
R=/tmp/r2p_reps
mkdir -p $R
$NCU -k regex:is_linreg_kernel -s 1 -c 1 -o $R/linreg python tools/prof_is.py linreg 1000000000 2 > $OUT/ncu_linreg.log 2>&1
$NCU -k regex:is_poly_kernel -s 1 -c 1 -o $R/poly python tools/prof_is.py poly 2000000000 2 > $OUT/ncu_poly.log 2>&1
$NCU -k regex:smc_resample_kernel -s 20 -c 1 -o $R/smc_k6 python tools/smc_time.py 100000000 30 > $OUT/ncu_k6.log 2>&1
$NCU -k regex:smc_scan_kernel -s 20 -c 1 -o $R/smc_k5 python tools/smc_time.py 100000000 30 > $OUT/ncu_k5.log 2>&1
$NCU -k regex:mh_gmm_kernel -s 0 -c 1 -o $R/mh python tools/prof_mh.py 4096 1000 1 > $OUT/ncu_mh.log 2>&1
$NCU -k regex:rs_ -s 3 -c 3 -o $R/resample python bench.py --workload resample --steps 1 --warmup 1 --no-cpu-baseline > $OUT/ncu_rs.log 2>&1
python tools/ncu_summary.py r2 $R/*.ncu-rep > $OUT/summary.log 2>&1
cp profiles/r2_ncu_summary.json $OUT/ 2>/dev/null
for f in $R/*.ncu-rep; do
  b=$(basename $f .ncu-rep)
  ncu -i $f --page source --csv --print-source sass > $R/$b.src.csv 2>/dev/null
  python tools/sass_mix.py $R/$b.src.csv > $OUT/sass_mix_$b.txt 2>&1
done
ls -la $OUT
