O=gpurun_out/polyc; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_is.py tests/test_gpu_scale.py -x -q -m gpu -k "poly or c5 or C5 or fig" > $O/tests.log 2>&1
for k in 1 2; do timeout 300 python bench.py --workload poly --steps 10 --warmup 3 --no-cpu-baseline > $O/p$k.json 2> $O/p$k.err; done
