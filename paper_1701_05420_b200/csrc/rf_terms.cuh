// Compile-time term tables of the factored order-m recursion (shared by
// recursion_fact.cu and recursion_stream.cu): terms are the subsets S of the
// modes {0..M-1} holding mode 0 with 2 <= |S| <= M-2, in mask order.
#pragma once

namespace bcg {

namespace rf {

__host__ __device__ constexpr int popc(int x) { return x == 0 ? 0 : (x & 1) + popc(x >> 1); }
__host__ __device__ constexpr int ipow(int b, int e) { return e == 0 ? 1 : b * ipow(b, e - 1); }

// terms: subsets S of {0..M-1} containing mode 0, 2 <= |S| <= M-2, by mask order
__host__ __device__ constexpr int term_count(int M) {
  int c = 0;
  for (int s = 1; s < (1 << M); s += 2)
    if (popc(s) >= 2 && popc(s) <= M - 2) ++c;
  return c;
}
__host__ __device__ constexpr int term_mask(int M, int t) {
  for (int s = 1; s < (1 << M); s += 2)
    if (popc(s) >= 2 && popc(s) <= M - 2) {
      if (t == 0) return s;
      --t;
    }
  return 0;
}
// row-major stride of mode q inside the factor block over the modes in `mask`
__host__ __device__ constexpr int stride_in(int mask, int q, int B) {
  int later = 0;
  for (int p = q + 1; p < 16; ++p)
    if (mask & (1 << p)) ++later;
  return ipow(B, later);
}
// compile-time offset contributed by the leading (register row) modes
// 0..M-CT-1 for row index `row` (row-major)
__host__ __device__ constexpr int head_offset(int mask, int M, int CT, int B, int row) {
  int off = 0;
  for (int q = M - CT - 1; q >= 0; --q) {
    const int digit = row % B;
    row /= B;
    if (mask & (1 << q)) off += digit * stride_in(mask, q, B);
  }
  return off;
}

// the same, forced to a compile-time constant (keeps the unrolled row loops
// cheap to compile: the offsets are folded by the front end)
template <int MASK, int M, int CT, int B, int ROW>
struct HeadOff {
  static constexpr int value = head_offset(MASK, M, CT, B, ROW);
};

}  // namespace rf

}  // namespace bcg
