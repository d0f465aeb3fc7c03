mkdir -p gpurun_out/r2l
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2l/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2l/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/r2l/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2l/smoke.log 2>&1
for w in linreg poly; do timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/r2l/$w.json 2> gpurun_out/r2l/$w.err; done
