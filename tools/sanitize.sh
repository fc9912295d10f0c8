#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py (under gpurun): bash tools/sanitize.sh <tag>
T=${1:-r02}
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py > gpurun_out/${T}_sanitize_${tool}.log 2>&1
  echo "$tool rc=$?"
done
