python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_smc.py -x -q 2>&1 | grep -E "^E |passed|failed" | head -3
timeout 300 python tools/smc_time.py 100000000 100
for mb in 4; do
python -c "
from paper_2010_08454_b200 import build as b
b.NVCC_FLAGS.append('-DCUPPL_SMC_MINBLOCKS=$mb')
b.build()"
echo "minblocks $mb"; timeout 300 python tools/smc_time.py 100000000 100
done
