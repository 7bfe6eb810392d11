// Shared device helpers of the moment kernel.
#pragma once

// Opt-in device bounds checks (build with -DBCG_CHECKS; see _build.py debug=True).
#ifdef BCG_CHECKS
#include <cstdio>
#define BCG_CHECK(cond, msg, v)                                                                \
  do {                                                                                         \
    if (!(cond)) {                                                                             \
      printf("BCG_CHECK %s:%d %s (value %lld) block %d thread %d\n", __FILE__, __LINE__, msg, \
             (long long)(v), (int)blockIdx.x, (int)threadIdx.x);                              \
      __trap();                                                                                \
    }                                                                                          \
  } while (0)
#else
#define BCG_CHECK(cond, msg, v) \
  do {                          \
  } while (0)
#endif
