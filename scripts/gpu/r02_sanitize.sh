# compute-sanitizer sweep over every kernel family (scripts/sanitize_case.py): tiny + ragged + vocab-tail configs
export PYTHONUNBUFFERED=1
for tool in memcheck synccheck racecheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 30 python scripts/sanitize_case.py all > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|SANITIZE_CASE_DONE" gpurun_out/san_$tool.log | tail -3
done
