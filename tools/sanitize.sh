#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over the kernel paths
# (tools/sanitize_case.py).  Output: gpurun_out/sanitize/<tool>_<case>.txt
set -u
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for c in "tiny" "ragged" "g8" "ragged fused" "config2"; do
    tag=$(echo "$c" | tr ' ' '_')
    extra=""
    [ "$tool" = "initcheck" ] && extra=""
    timeout ${SAN_TIMEOUT:-600} $CS --tool $tool $extra --print-limit 20 python tools/sanitize_case.py $c \
      > gpurun_out/sanitize/${tool}_${tag}.txt 2>&1
    echo "$tool $tag rc=$? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|OK max_abs' gpurun_out/sanitize/${tool}_${tag}.txt | tr '\n' ' ')"
  done
done
