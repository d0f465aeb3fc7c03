OUT=gpurun_out/r2z
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for i in 1 2; do timeout 600 python bench.py --workload poly --no-cpu-baseline > $OUT/poly$i.json 2>&1; done
timeout 600 python bench.py --workload linreg --no-cpu-baseline > $OUT/linreg.json 2>&1
