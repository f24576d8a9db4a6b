#!/bin/bash
# The GPU test suite against the checked build (device-side invariant checks,
# csrc/rsv_check.h) -- the stand-in for compute-sanitizer, which is closed on
# this pool.  Usage (on the GPU box): bash tools/checked_run.sh [pytest args]
set -o pipefail
mkdir -p gpurun_out
[ -f paper_1603_08114_b200/librsvhmc_b200_checked.so ] || make -s -C paper_1603_08114_b200/csrc checked
RSV_LIB=checked python -m pytest tests -m gpu -q -p no:cacheprovider "$@" 2>&1 | tee gpurun_out/checked_run.log
