mkdir -p gpurun_out
timeout 900 python scripts/append_ab.py 2>&1 | grep AB
for tool in memcheck synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tests/sanitize_run.py > gpurun_out/r2b_sanitize_$tool.txt 2>&1
  echo "$tool exit $?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|SANITIZE_RUN|FAIL" gpurun_out/r2b_sanitize_$tool.txt | tail -4
done
