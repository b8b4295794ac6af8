for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 200 python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_$tool.log
  echo "== $tool"; grep "SUMMARY\|family\|ok \[" gpurun_out/sanitize_$tool.log | tail -14
  grep "^=========     at " gpurun_out/sanitize_$tool.log | sed 's/+0x[0-9a-f]*//' | sort | uniq -c | head
done
