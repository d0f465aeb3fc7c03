for st in 4 16 2; do
python -c "
from paper_2010_08454_b200 import build as b
b.NVCC_FLAGS.append('-DCUPPL_SCAN_TILES=$st')
b.build()"
echo "scan tiles $st"
python tools/smc_time.py 100000000 100 | cut -c1-80
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:smc_scan -c 5 python tools/smc_time.py 100000000 10 2>/dev/null | grep smc_scan | tail -1 | awk -F, '{print $NF}'
done
