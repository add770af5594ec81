# compute-sanitizer over tests/sanitize_run.py; summaries to gpurun_out/
mkdir -p gpurun_out
timeout 300 python tests/sanitize_run.py > gpurun_out/sanitize_plain.txt 2>&1; tail -2 gpurun_out/sanitize_plain.txt
for tool in memcheck synccheck initcheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tests/sanitize_run.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool exit $?"; grep -E "ERROR SUMMARY|SANITIZE_RUN|Error|error" gpurun_out/sanitize_$tool.txt | tail -4
done
