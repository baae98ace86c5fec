for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 30 python tools/sanitize_cases.py ${CASES:-k1_fused k1_split k1_fused_table k1_split_table} > gpurun_out/san2_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|case ok" gpurun_out/san2_$tool.log | tr '\n' ' '; echo
done
