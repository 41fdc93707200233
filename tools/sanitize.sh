#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over one small
# invocation of every kernel family (tools/sanitize_run.py); run under gpurun.
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout -s KILL 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 \
    python tools/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/sanitize_$tool.log
done
