for cfg in "16 4" "32 3" "32 4" "32 2"; do
set -- $cfg
python -c "
from paper_2010_08454_b200 import build as b
b.NVCC_FLAGS += ['-DCUPPL_K6_SRC=$1', '-DCUPPL_SMC_MINBLOCKS=$2']
b.build()"
echo "src $1 minblocks $2"
timeout 600 python -m pytest tests/test_gpu_smc.py -q -x 2>&1 | grep -E "^FAILED|passed|failed" | head -2
timeout 300 python tools/smc_time.py 100000000 100 | cut -c1-90
done
