# One bench line per workload (default config of each) + the reference arm, saved under gpurun_out/bench/.
mkdir -p gpurun_out/bench
python -c "import __graft_entry__ as g; g.build()"
for w in linreg poly smc mh dsl-linreg; do
  timeout 900 python bench.py --workload $w > gpurun_out/bench/$w.json 2> gpurun_out/bench/$w.err
  timeout 600 python bench.py --workload $w --impl reference --steps 2 --warmup 1 > gpurun_out/bench/ref_$w.json 2>> gpurun_out/bench/$w.err
done
tail -n 2 gpurun_out/bench/*.err
