#!/bin/bash
# compute-sanitizer over tools/sanitize_driver.py (every kernel family, ragged tails)
mkdir -p gpurun_out
python tools/sanitize_driver.py > gpurun_out/sanitize_plain.log 2>&1; echo "plain rc=$?" >> gpurun_out/sanitize_plain.log
for T in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $T --target-processes all python tools/sanitize_driver.py > gpurun_out/sanitize_$T.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$T.log
done
