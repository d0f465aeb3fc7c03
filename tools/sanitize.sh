# compute-sanitizer over smoke() (every engine: IS poly/linreg, SMC K4-K6, MH K7, a compiled
# CuPPL model) with each tool; summaries under gpurun_out/sanitize/ (SURVEY.md §4 item 5).
OUT=gpurun_out/sanitize
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()"
SM="${SANITIZE_CMD:-python -c 'import __graft_entry__ as g; g.smoke()'}"
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  extra=""
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 30 bash -c "$SM" > $OUT/$tool.log 2>&1
  echo "$tool exit=$?"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|smoke |sanitize_extra" $OUT/$tool.log | tail -8
done
