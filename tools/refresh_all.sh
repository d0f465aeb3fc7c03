# Round-end refresh: every bench line (ours + reference arm), one `ncu --set full` per dominant
# kernel, launch lists; outputs under gpurun_out/{bench,prof,prof_dsl}.
bash tools/bench_all.sh
bash tools/profile_all.sh
NCU="ncu --set full --import-source on --clock-control none -f"
$NCU -k regex:cuppl_dsl_model -s 2 -c 1 -o gpurun_out/prof/dsl_linreg \
  python bench.py --workload dsl-linreg --steps 1 --warmup 1 --no-cpu-baseline --particles 200000000 > gpurun_out/prof/dsl.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_dsl_linreg.csv \
  python bench.py --workload dsl-linreg --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/prof gpurun_out/bench
