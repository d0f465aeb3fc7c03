OUT=gpurun_out/r2q
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_resample.py tests/test_gpu_smc.py -q -x > $OUT/tests.log 2>&1
echo "rc=$?" >> $OUT/tests.log
for w in smc resample; do
  timeout 900 python bench.py --workload $w > $OUT/bench_$w.json 2> $OUT/bench_$w.err
  timeout 600 python bench.py --workload $w --impl reference --steps 2 --warmup 1 > $OUT/ref_$w.json 2>> $OUT/bench_$w.err
done
L="ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
$L -c 400 --log-file $OUT/launches_smc.csv python tools/smc_time.py 100000000 100 > /dev/null 2>&1
$L --log-file $OUT/launches_resample.csv python bench.py --workload resample --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
NCU="ncu --set full --import-source on --clock-control none -f"
R=/tmp/r2q_reps
mkdir -p $R
$NCU -k regex:smc_resample_kernel -s 20 -c 1 -o $R/smc_k6 python tools/smc_time.py 100000000 30 > $OUT/ncu_k6.log 2>&1
$NCU -k regex:smc_scan_kernel -s 20 -c 1 -o $R/smc_k5 python tools/smc_time.py 100000000 30 > $OUT/ncu_k5.log 2>&1
$NCU -k regex:rs_ -s 3 -c 3 -o $R/resample python bench.py --workload resample --steps 1 --warmup 1 --no-cpu-baseline > $OUT/ncu_rs.log 2>&1
python tools/ncu_summary.py r2q $R/*.ncu-rep > $OUT/summary.log 2>&1
cp profiles/r2q_ncu_summary.json $OUT/ 2>/dev/null
for f in $R/*.ncu-rep; do
  b=$(basename $f .ncu-rep)
  ncu -i $f --page source --csv --print-source sass > $R/$b.src.csv 2>/dev/null
  python tools/sass_mix.py $R/$b.src.csv > $OUT/sass_mix_$b.txt 2>&1
done
