set -x
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()"
python tools/prof_is.py poly 12500000000 4
ncu --set full --import-source on --clock-control none -k regex:is_poly_kernel -s 1 -c 1 -f -o $OUT/poly python tools/prof_is.py poly 2000000000 2 > $OUT/prof_is.log 2>&1
tail -2 $OUT/prof_is.log
