#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck of tools/sanitize_run.py (run under gpurun)
out=gpurun_out/sanitizer.txt
echo "# compute-sanitizer on tools/sanitize_run.py 300, one B200" > $out
for tool in memcheck racecheck synccheck; do
  echo "## $tool" >> $out
  timeout 1500 compute-sanitizer --tool $tool python tools/sanitize_run.py 300 2>&1 | grep -E "COMPUTE-SANITIZER|ERROR SUMMARY|RACECHECK SUMMARY|SYNCCHECK|sanitize run ok|Error|error" | head -20 >> $out
done
cat $out
