# The compiled-model workload (dsl-linreg): bench line, one `ncu --set full` capture of the
# NVRTC kernel (cuppl_dsl_model) and the launch list of the bench command.
set -x
OUT=gpurun_out/prof_dsl
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python bench.py --workload dsl-linreg > $OUT/bench_dsl.json 2> $OUT/bench_dsl.err
ncu --set full --import-source on --clock-control none -f -k regex:cuppl_dsl_model -s 2 -c 1 -o $OUT/dsl_linreg \
  python bench.py --workload dsl-linreg --steps 1 --warmup 1 --no-cpu-baseline --particles 200000000 > $OUT/ncu.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_dsl.csv \
  python bench.py --workload dsl-linreg --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ls -la $OUT
