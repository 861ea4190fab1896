#!/bin/bash
mkdir -p gpurun_out
for c in ${CASES:-pair:racecheck pair:memcheck p2p:memcheck p2p:racecheck conv:memcheck conv:racecheck}; do
  case=${c%%:*}; tool=${c##*:}
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py $case > gpurun_out/sanitize_${case}_${tool}.log 2>&1
  echo "sanitize $case $tool rc=$?"; tail -2 gpurun_out/sanitize_${case}_${tool}.log
done
