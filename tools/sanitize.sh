#!/bin/bash
# compute-sanitizer, one tool per call (B200_PROFILING.md): bash tools/sanitize.sh <tool>
# Runs tools/sanitize_run.py under both launch schedules and the opt-in k-split kernel; logs to gpurun_out/.
tool=$1
python tools/sanitize_run.py > gpurun_out/san_plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/san_plain.log; exit 1; }
for env in "SFMG_EARLY_MAXN=0" "SFMG_EARLY_MAXN=16777216" "SFMG_KSPLIT=1"; do
  echo "== $tool $env" >> gpurun_out/sanitize_$tool.log
  env $env timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py >> gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.log
done
grep -E "^==|ERROR SUMMARY|RACECHECK SUMMARY|rc=|Program hit" gpurun_out/sanitize_$tool.log
