mkdir -p gpurun_out/r2a
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2a/smoke.log 2>&1
nvidia-smi > gpurun_out/r2a/smi.txt; nproc >> gpurun_out/r2a/smi.txt; free -g >> gpurun_out/r2a/smi.txt
for w in linreg poly smc mh; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/r2a/$w.json 2> gpurun_out/r2a/$w.err
done
