// Dense-entry verification kernel (SURVEY §8 f row 4: a GPU dense oracle for
// verification beyond the reference's n^m <= 1e8 dense oracle,
// bc/oracle.py:22-34, 89-117).
//
// For E element tuples (i_1..i_m) of the order-m tensor (any order of the
// indices, repeats allowed), one pass over the samples accumulates the raw
// product sums of ALL 2^m sub-tuples of the centered data:
//
//   P[e][S] = sum_l prod_{q in S} (x[l, i_q] - mean[i_q]),   S subset of {0..m-1}
//
// (P[e][0] = t).  It shares nothing with the product path -- no block layout,
// no Khatri-Rao GEMM, no packed tensors, no recursion -- so the cumulants the
// host forms from P by the moment-cumulant formula over set partitions
// (verify.py) are an independent check of cumulants_upto at full size.
//
// Work split: grid (E, P); block p of entry e sums the samples l = p, p + P,
// ...  (strided), each thread a fixed sample stride; the 2^m products of one
// sample are formed incrementally (prod[S] = prod[S minus its top bit] *
// x[top]); the block reduces its threads in a fixed tree and the second pass
// adds the P partials in order -- deterministic.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace bcg {

constexpr int kDenseThreads = 128;

template <int M>
__global__ void __launch_bounds__(kDenseThreads) k_dense_subsets(const double *__restrict__ x, int64_t t, int64_t n,
                                                                  int64_t ldx, const double *__restrict__ mean,
                                                                  const int32_t *__restrict__ idx,
                                                                  double *__restrict__ part) {
  constexpr int NS = 1 << M;
  const int e = blockIdx.x, p = blockIdx.y, P = gridDim.y;
  int col[M];
  double mu[M];
#pragma unroll
  for (int q = 0; q < M; ++q) {
    col[q] = idx[(int64_t)e * M + q];
    mu[q] = mean[col[q]];
  }
  double acc[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) acc[s] = 0.0;
  for (int64_t l = (int64_t)p * kDenseThreads + threadIdx.x; l < t; l += (int64_t)P * kDenseThreads) {
    const double *row = x + l * ldx;
    double v[M];
#pragma unroll
    for (int q = 0; q < M; ++q) v[q] = row[col[q]] - mu[q];
    double prod[NS];
    prod[0] = 1.0;
#pragma unroll
    for (int s = 1; s < NS; ++s) {
      const int top = 31 - __clz(s);
      prod[s] = prod[s ^ (1 << top)] * v[top];
    }
#pragma unroll
    for (int s = 1; s < NS; ++s) acc[s] += prod[s];
  }
  // fixed-order tree over the block's threads, one subset at a time
  __shared__ double red[kDenseThreads];
  for (int s = 1; s < NS; ++s) {
    red[threadIdx.x] = acc[s];
    __syncthreads();
    for (int w = kDenseThreads / 2; w > 0; w >>= 1) {
      if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x == 0) part[((int64_t)e * P + p) * NS + s] = red[0];
    __syncthreads();
  }
}

__global__ void k_dense_reduce(const double *__restrict__ part, int64_t E, int P, int NS, int64_t t,
                               double *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E * NS; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i / NS;
    const int s = (int)(i % NS);
    if (s == 0) {
      out[i] = (double)t;
      continue;
    }
    double v = 0.0;
    for (int p = 0; p < P; ++p) v += part[(e * P + p) * NS + s];
    out[i] = v;
  }
}

int dense_subsets_parts(int64_t E, int64_t t) {
  // about 4 waves of 148 SMs over all entries, at least 1 block per entry,
  // at most one block per 128 samples
  int64_t P = (148 * 16 + E - 1) / (E > 0 ? E : 1);
  const int64_t pmax = (t + kDenseThreads - 1) / kDenseThreads;
  if (P > pmax) P = pmax;
  if (P > 1024) P = 1024;
  return (int)(P < 1 ? 1 : P);
}

cudaError_t launch_dense_subsets(const double *x, int64_t t, int64_t n, int64_t ldx, const double *mean, int m,
                                 const int32_t *idx, int64_t E, double *part, int P, double *out,
                                 cudaStream_t stream) {
  if (E <= 0) return cudaSuccess;
  const dim3 grid((unsigned)E, (unsigned)P);
  switch (m) {
#define DS(M) \
  case M: k_dense_subsets<M><<<grid, kDenseThreads, 0, stream>>>(x, t, n, ldx, mean, idx, part); break;
    DS(1) DS(2) DS(3) DS(4) DS(5) DS(6) DS(7) DS(8)
#undef DS
    default: return cudaErrorInvalidValue;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  g_launches++;
  const int NS = 1 << m;
  int64_t blocks = (E * NS + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_dense_reduce<<<(unsigned)blocks, 256, 0, stream>>>(part, E, P, NS, t, out);
  g_launches++;
  return cudaGetLastError();
}

}  // namespace bcg
