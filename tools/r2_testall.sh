# Round-2 validation pass: the whole -m gpu suite, smoke(), compute-sanitizer over smoke() and
# tools/sanitize_extra.py. Outputs under gpurun_out/r2_testall/.
OUT=gpurun_out/r2_testall
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
echo "smoke rc=$?" >> $OUT/smoke.log
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 30 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/san_smoke_$tool.log 2>&1
  timeout 1200 compute-sanitizer --tool $tool --print-limit 30 python tools/sanitize_extra.py > $OUT/san_extra_$tool.log 2>&1
done
grep -h "ERROR SUMMARY\|RACECHECK SUMMARY\|smoke \|sanitize_extra" $OUT/san_*.log > $OUT/sanitize_summary.txt
