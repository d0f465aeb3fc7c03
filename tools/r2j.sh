mkdir -p gpurun_out/r2j
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2j/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_is.py tests/test_program.py -q -x > gpurun_out/r2j/is.log 2>&1
timeout 600 python bench.py --workload linreg --no-cpu-baseline --particles 100000000 --steps 3 > gpurun_out/r2j/lin.json 2>&1
python - > gpurun_out/r2j/bigD.log 2>&1 <<'PY'
import torch, time
from paper_2010_08454_b200 import Rng, infer, models
for D in (1000, 3968, 10000, 100000):
    m = models.LinearRegression.synthetic(n_points=D)
    la = infer.IsLauncher(m)
    n = 100_000_000 if D <= 10000 else 10_000_000
    la.launch(0, n, 1); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); la.launch(0, n, 2); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(D, n, ms, "particle-points/s %.3g" % (n * D / (ms / 1e3)))
PY
