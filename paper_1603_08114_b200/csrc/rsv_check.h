// rsv_check.h -- device-side invariant checks of the checked build
// (make checked -> librsvhmc_b200_checked.so, RSV_LIB selects it).  The
// checks guard the indices the kernels compute themselves: staging windows
// and their alignment (bulk copies), shared-memory slots, window and record
// capacities, parse-queue bounds.  compute-sanitizer is closed on this GPU
// pool (profiles/r02_compute_sanitizer_refused.log); the checked build runs
// the GPU test suite instead (tools/checked_run.sh).  A failed check prints
// file:line and the condition, then traps (the launch fails with an error).
#pragma once
#include <stdio.h>

#ifdef RSV_CHECKED
#define RSV_CHECK(cond)                                                                        \
  do {                                                                                         \
    if (!(cond)) {                                                                             \
      printf("RSV_CHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, (int)blockIdx.x, \
             (int)threadIdx.x, #cond);                                                         \
      __trap();                                                                                \
    }                                                                                          \
  } while (0)
#else
#define RSV_CHECK(cond) \
  do {                  \
  } while (0)
#endif
