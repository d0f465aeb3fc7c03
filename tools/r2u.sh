OUT=gpurun_out/r2u
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_resample.py -q -x > $OUT/tests.log 2>&1
echo "rc=$?" >> $OUT/tests.log
timeout 600 python bench.py --workload resample --no-cpu-baseline > $OUT/resample.json 2>&1
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv -k regex:"rs_" -c 6 --log-file $OUT/k.csv python bench.py --workload resample --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 600 compute-sanitizer --tool memcheck python -c "
import torch
from paper_2010_08454_b200 import resample, Rng
g = torch.Generator(device='cuda').manual_seed(0)
for n in (1, 2048, 2049, 70001):
    lw = torch.randn(n, device='cuda', generator=g)
    for pay in (None, torch.arange(n, dtype=torch.int32, device='cuda'), torch.randn((n, 4), device='cuda', generator=g), torch.zeros((n, 5), dtype=torch.uint8, device='cuda'), torch.randn((n, 16), device='cuda', generator=g)):
        resample.systematic(lw, pay, Rng(8), 1, ancestors=True)
torch.cuda.synchronize(); print('ok')
" > $OUT/memcheck.log 2>&1
timeout 600 compute-sanitizer --tool racecheck python -c "
import torch
from paper_2010_08454_b200 import resample, Rng
g = torch.Generator(device='cuda').manual_seed(0)
for n in (2049, 70001):
    lw = torch.randn(n, device='cuda', generator=g)
    resample.systematic(lw, torch.arange(n, dtype=torch.int32, device='cuda'), Rng(8), 1, ancestors=True)
torch.cuda.synchronize(); print('ok')
" > $OUT/racecheck.log 2>&1
