#!/bin/bash
# compute-sanitizer over the blend kernels (K3/K4/K3x/K4x and the binning
# pipeline) on a small scene; logs -> gpurun_out/sanitize_<tool>.log
for t in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_case.py \
    > gpurun_out/sanitize_$t.log 2>&1
  echo "$t rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_$t.log | tail -1)"
done
