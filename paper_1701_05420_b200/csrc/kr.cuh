// Khatri-Rao factor of one sample row: prod_{q < NQ} xr[cols[q]].
// NQ > 0: compile-time mode count (exactly NQ-1 DMULs, no predication);
// NQ == 0: runtime count nq (orders m > 8, generic path).
#pragma once

namespace bcg {

// ONES: column index -1 denotes the constant-ones column of a fused
// multi-order plan (factor 1.0; no load).
template <bool ONES>
__device__ __forceinline__ double kr_val(const double *xr, int c) {
  if constexpr (ONES) {
    const double v = xr[c < 0 ? 0 : c];
    return c < 0 ? 1.0 : v;
  } else {
    return xr[c];
  }
}

template <int NQ, bool ONES = false>
__device__ __forceinline__ double kr_prod(const double *xr, const int (&cols)[8], int nq) {
  double p = kr_val<ONES>(xr, cols[0]);
  if constexpr (NQ > 0) {
#pragma unroll
    for (int q = 1; q < NQ; ++q) p *= kr_val<ONES>(xr, cols[q]);
  } else {
#pragma unroll
    for (int q = 1; q < 8; ++q)
      if (q < nq) p *= kr_val<ONES>(xr, cols[q]);
  }
  return p;
}

// instantiate `FN<..., M>` for the orders with compile-time mode counts
#define BCG_DISPATCH_M(m, FN, ...)      \
  switch (m) {                           \
    case 2: FN(2, __VA_ARGS__); break;   \
    case 3: FN(3, __VA_ARGS__); break;   \
    case 4: FN(4, __VA_ARGS__); break;   \
    case 5: FN(5, __VA_ARGS__); break;   \
    case 6: FN(6, __VA_ARGS__); break;   \
    case 7: FN(7, __VA_ARGS__); break;   \
    case 8: FN(8, __VA_ARGS__); break;   \
    default: FN(0, __VA_ARGS__); break;  \
  }

}  // namespace bcg

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
