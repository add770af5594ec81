mkdir -p gpurun_out
for tool in synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tests/sanitize_run.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool exit $?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|SANITIZE_RUN" gpurun_out/sanitize_$tool.txt | tail -3
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "batch_run_snapshot or cluster_merge or flash_query_batch" 2>&1 | tail -2
python scripts/qkv_trace.py 2>&1 | tail -20
