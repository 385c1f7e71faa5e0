#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the shipped kernels (tools/sanitize_case.py),
# plus memcheck of the GA / scene kernel tests.  Logs: gpurun_out/sanitize_<tool>_<case>.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for c in tiny_forward attention_kvsplit ring_merge camera_head_1b agg1b_s2; do
    if [ "$tool" != memcheck ] && [ "$c" = agg1b_s2 ]; then continue; fi
    timeout ${SAN_TIMEOUT:-600} $CS --tool $tool --error-exitcode 99 --print-limit 20 \
      python tools/sanitize_case.py $c > gpurun_out/sanitize_${tool}_${c}.log 2>&1
    echo "$tool $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|: ok' gpurun_out/sanitize_${tool}_${c}.log | tr '\n' ' ')"
  done
done
timeout ${SAN_TIMEOUT:-900} $CS --tool memcheck --error-exitcode 99 --print-limit 20 \
  python -m pytest tests/test_ga.py tests/test_scene.py tests/test_epipolar.py -m gpu -q -x -p no:cacheprovider \
  > gpurun_out/sanitize_memcheck_ga_scene.log 2>&1
echo "memcheck ga/scene/epipolar tests rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/sanitize_memcheck_ga_scene.log | tail -2 | tr '\n' ' ')"
