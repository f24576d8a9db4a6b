#!/bin/bash
# compute-sanitizer over the GPU parity tests at small sizes (run on the GPU box):
#   racecheck (shared-memory hazards), synccheck (barrier / mbarrier use),
#   memcheck (out-of-bounds / misaligned global and shared accesses),
#   initcheck (reads of uninitialised device memory).
# Logs -> gpurun_out/sanitize_<tool>.log; per-tool wall limit $1 seconds (default 1500).
LIM=${1:-1500}
mkdir -p gpurun_out
SEL='not 3000017 and not 1048576 and not 100003 and not large_T and not zero_copy and not long_trajectory'
FILES="tests/test_gpu_parity.py tests/test_gpu_ensemble.py tests/test_gpu_blocked.py tests/test_gpu_robustness.py"
for tool in ${TOOLS:-memcheck synccheck racecheck initcheck}; do
  extra=""
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  [ "$tool" = initcheck ] && extra="--track-unused-memory no"
  timeout $LIM compute-sanitizer --tool $tool $extra --print-limit 50 --error-exitcode 99 \
    python -m pytest $FILES -m gpu -q -x -k "$SEL" -p no:cacheprovider > gpurun_out/sanitize_$tool.log 2>&1
  echo "exit $?" >> gpurun_out/sanitize_$tool.log
done
