// K1: column statistics, finite scan and centering (bc/moments.py:23-41,
// bc/cumulants.py:31-39), plus small packed-buffer helpers.  All HBM-bound;
// reductions are two-pass with a fixed order (no float atomics), so results
// are bitwise reproducible.
#include <cuda_runtime.h>

#include <climits>
#include <algorithm>
#include <cstdint>

#include "kernels.h"

namespace bcg {

constexpr int kCsThreads = 256;

// Pass 1: partition p sums rows [p*t/P, (p+1)*t/P) of every column.
__global__ void __launch_bounds__(kCsThreads)
    k_colstats_partial(const double *__restrict__ x, int64_t t, int64_t n, int64_t ldx, int nparts,
                       double *__restrict__ part_sum, double *__restrict__ part_sq,
                       unsigned long long *first_bad) {
  __shared__ double red_s[kCsThreads], red_q[kCsThreads];
  const int p = blockIdx.x;
  const int64_t r0 = t * p / nparts, r1 = t * (p + 1) / nparts;
  const int tid = threadIdx.x;
  const int lanes = n < kCsThreads ? (int)n : kCsThreads;  // threads per row
  const int rpi = kCsThreads / lanes;                      // rows per iteration
  const int c0 = tid % lanes, rph = tid / lanes;
  const bool active = rph < rpi;
  for (int64_t cbase = 0; cbase < n; cbase += lanes) {
    const int64_t c = cbase + c0;
    double s = 0.0, q = 0.0;
    if (active && c < n) {
      unsigned long long bad = ~0ULL;  // first non-finite position seen (one atomic per thread, after the loop)
#pragma unroll 4
      for (int64_t r = r0 + rph; r < r1; r += rpi) {
        const double v = x[r * ldx + c];
        if (!isfinite(v)) bad = min(bad, (unsigned long long)(r * n + c));
        s += v;
        q += v * v;
      }
      if (bad != ~0ULL) atomicMin(first_bad, bad);
    }
    red_s[tid] = s;
    red_q[tid] = q;
    __syncthreads();
    if (rph == 0 && c < n) {
      double ss = 0.0, qq = 0.0;
      for (int k = 0; k < rpi; ++k) {
        ss += red_s[k * lanes + c0];
        qq += red_q[k * lanes + c0];
      }
      part_sum[(int64_t)p * n + c] = ss;
      part_sq[(int64_t)p * n + c] = qq;
    }
    __syncthreads();
  }
}

// Pass 2: ordered sum over partitions.
__global__ void k_colstats_final(const double *__restrict__ part_sum, const double *__restrict__ part_sq,
                                 int nparts, int64_t n, int64_t t, double *sums, double *mean, double *sumsq,
                                 unsigned long long *first_bad) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0, q = 0.0;
    for (int p = 0; p < nparts; ++p) {
      s += part_sum[(int64_t)p * n + c];
      q += part_sq[(int64_t)p * n + c];
    }
    if (sums) sums[c] = s;
    if (mean) mean[c] = s / (double)t;
    if (sumsq) sumsq[c] = q;
  }
  if (first_bad && blockIdx.x == 0 && threadIdx.x == 0) {
    if (*first_bad >= 0x7F7F7F7F7F7F7F7FULL) *reinterpret_cast<long long *>(first_bad) = -1;
  }
}

int colstats_parts(int64_t t, int64_t n) {
  (void)n;
  int64_t parts = (t + 255) / 256;
  if (parts > 148 * 4) parts = 148 * 4;
  if (parts < 1) parts = 1;
  return (int)parts;
}

cudaError_t launch_colstats(const double *x, int64_t t, int64_t n, int64_t ldx, double *sums, double *mean,
                            double *sumsq, int64_t *first_bad, double *scratch, int nparts,
                            cudaStream_t stream) {
  unsigned long long *fb = reinterpret_cast<unsigned long long *>(first_bad);
  unsigned long long *fb_scratch = reinterpret_cast<unsigned long long *>(scratch + 2 * (int64_t)nparts * n);
  if (!fb) fb = fb_scratch;
  cudaError_t e = cudaMemsetAsync(fb, 0x7F, sizeof(unsigned long long), stream);
  if (e != cudaSuccess) return e;
  k_colstats_partial<<<nparts, kCsThreads, 0, stream>>>(x, t, n, ldx, nparts, scratch, scratch + (int64_t)nparts * n,
                                                         fb);
  g_launches++;
  int blocks = (int)((n + 255) / 256);
  k_colstats_final<<<blocks, 256, 0, stream>>>(scratch, scratch + (int64_t)nparts * n, nparts, n, t, sums, mean,
                                               sumsq, first_bad ? fb : nullptr);
  g_launches++;
  return cudaGetLastError();
}

// xc = x - mean, one warp per row, lanes across columns (coalesced).
__global__ void k_center(const double *__restrict__ x, int64_t t, int64_t n, int64_t ldx,
                         const double *__restrict__ mean, double *__restrict__ xc) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < t; r += nwarps)
    for (int64_t c = lane; c < n; c += 32) xc[r * n + c] = x[r * ldx + c] - mean[c];
}

cudaError_t launch_center(const double *x, int64_t t, int64_t n, int64_t ldx, const double *mean, double *xc,
                          cudaStream_t stream) {
  int64_t blocks = (t + 7) / 8;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  k_center<<<(int)blocks, 256, 0, stream>>>(x, t, n, ldx, mean, xc);
  g_launches++;
  return cudaGetLastError();
}

// x[l, c] = xt[c, l]  (reference passes the transposed data, bc/_engines.py:95)
__global__ void k_transpose(const double *__restrict__ xt, int64_t n, int64_t t, double *__restrict__ x) {
  __shared__ double tile[32][33];
  const int64_t l0 = blockIdx.x * 32LL, c0 = blockIdx.y * 32LL;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t c = c0 + i, l = l0 + threadIdx.x;
    if (c < n && l < t) tile[i][threadIdx.x] = xt[c * t + l];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t l = l0 + i, c = c0 + threadIdx.x;
    if (c < n && l < t) x[l * n + c] = tile[threadIdx.x][i];
  }
}

cudaError_t launch_transpose(const double *xt, int64_t n, int64_t t, double *x, cudaStream_t stream) {
  dim3 grid((unsigned)((t + 31) / 32), (unsigned)((n + 31) / 32));
  k_transpose<<<grid, dim3(32, 8), 0, stream>>>(xt, n, t, x);
  g_launches++;
  return cudaGetLastError();
}

__global__ void k_axpby(int64_t len, double a, const double *x, double c, const double *y, double *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
    // two roundings each, no FMA contraction: the same float ops as numpy's
    // `v * s` and `u + w` (bc/symtensor.py:185-200)
    double v = __dmul_rn(a, x[i]);
    if (y) v = __dadd_rn(v, __dmul_rn(c, y[i]));
    out[i] = v;
  }
}

cudaError_t launch_axpby(int64_t len, double a, const double *x, double c, const double *y, double *out,
                         cudaStream_t stream) {
  if (len <= 0) return cudaSuccess;
  int64_t blocks = (len + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_axpby<<<(int)blocks, 256, 0, stream>>>(len, a, x, c, y, out);
  g_launches++;
  return cudaGetLastError();
}

__global__ void k_div(int64_t len, const double *x, double d, double *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __ddiv_rn(x[i], d);
}

cudaError_t launch_div(int64_t len, const double *x, double d, double *out, cudaStream_t stream) {
  if (len <= 0) return cudaSuccess;
  int64_t blocks = (len + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_div<<<(int)blocks, 256, 0, stream>>>(len, x, d, out);
  g_launches++;
  return cudaGetLastError();
}

// xt[c, l] = x[l, c] - (mean ? mean[c] : 0) for l < t, 0 for t <= l < ldt:
// the padded transposed layout the moment kernel stages (32 x 32 smem tiles,
// coalesced on both sides).
__global__ void k_transpose_pad(const double *__restrict__ x, int64_t t, int64_t n, int64_t ldx,
                                const double *__restrict__ mean, double *__restrict__ xt, int64_t ldt) {
  __shared__ double tile[32][33];
  const int64_t l0 = blockIdx.x * 32LL, c0 = blockIdx.y * 32LL;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t l = l0 + i, c = c0 + threadIdx.x;
    double v = 0.0;
    if (l < t && c < n) v = x[l * ldx + c] - (mean ? mean[c] : 0.0);
    tile[i][threadIdx.x] = v;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t c = c0 + i, l = l0 + threadIdx.x;
    if (c < n && l < ldt) xt[c * ldt + l] = tile[threadIdx.x][i];
  }
}

cudaError_t launch_transpose_pad(const double *x, int64_t t, int64_t n, int64_t ldx, const double *mean, double *xt,
                                 int64_t ldt, cudaStream_t stream) {
  dim3 grid((unsigned)((ldt + 31) / 32), (unsigned)((n + 31) / 32));
  k_transpose_pad<<<grid, dim3(32, 8), 0, stream>>>(x, t, n, ldx, mean, xt, ldt);
  g_launches++;
  return cudaGetLastError();
}

// dst[c, l] = src[c, l] for l < t (src row stride lds), 0 up to ldt
__global__ void k_pad_rows(const double *__restrict__ src, int64_t n, int64_t t, int64_t lds, double *__restrict__ dst,
                           int64_t ldt) {
  const int64_t total = n * ldt;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i / ldt, l = i - c * ldt;
    dst[i] = l < t ? src[c * lds + l] : 0.0;
  }
}

cudaError_t launch_pad_rows(const double *src, int64_t n, int64_t t, int64_t lds, double *dst, int64_t ldt,
                            cudaStream_t stream) {
  int64_t blocks = (n * ldt + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  k_pad_rows<<<(int)blocks, 256, 0, stream>>>(src, n, t, lds, dst, ldt);
  g_launches++;
  return cudaGetLastError();
}

// per row c of xt (n x ldt): sums[c] = sum_{l<t} xt[c, l], sumsq[c] = sum xt^2.
// Segment p of P of each row per CTA (grid n x P, so even n = 36 fills the
// GPU), 4 loads in flight per thread, fixed-order tree; with P > 1 the
// partials go to `part` and k_rowstats_final adds them in segment order
// (deterministic).
__global__ void k_rowstats(const double *__restrict__ xt, int64_t t, int64_t ldt, int P, double *sums,
                           double *sumsq, double *__restrict__ part) {
  __shared__ double rs[256], rq[256];
  const int64_t c = blockIdx.x / P;
  const int p = blockIdx.x % P;
  const int64_t l0 = t * p / P, l1 = t * (p + 1) / P;
  double s = 0.0, q = 0.0;
  const double *row = xt + c * ldt;
#pragma unroll 4
  for (int64_t l = l0 + threadIdx.x; l < l1; l += 256) {
    const double v = row[l];
    s += v;
    q += v * v;
  }
  rs[threadIdx.x] = s;
  rq[threadIdx.x] = q;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      rs[threadIdx.x] += rs[threadIdx.x + w];
      rq[threadIdx.x] += rq[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (part) {
      part[2 * blockIdx.x] = rs[0];
      part[2 * blockIdx.x + 1] = rq[0];
    } else {
      if (sums) sums[c] = rs[0];
      if (sumsq) sumsq[c] = rq[0];
    }
  }
}

__global__ void k_rowstats_final(const double *__restrict__ part, int64_t n, int P, double *sums, double *sumsq) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0, q = 0.0;
    for (int p = 0; p < P; ++p) {
      s += part[2 * (c * P + p)];
      q += part[2 * (c * P + p) + 1];
    }
    if (sums) sums[c] = s;
    if (sumsq) sumsq[c] = q;
  }
}

int rowstats_parts(int64_t n, int64_t t) {
  int64_t P = (4 * 148 + n - 1) / n;
  const int64_t by_len = (t + 4095) / 4096;  // >= 4096 samples per segment
  if (P > by_len) P = by_len;
  return P < 1 ? 1 : (int)P;
}

cudaError_t launch_rowstats(const double *xt, int64_t n, int64_t t, int64_t ldt, double *sums, double *sumsq,
                            double *ws, int P, cudaStream_t stream) {
  if (!ws) P = 1;
  k_rowstats<<<(unsigned)(n * P), 256, 0, stream>>>(xt, t, ldt, P, sums, sumsq, P > 1 ? ws : nullptr);
  g_launches++;
  if (P > 1) {
    k_rowstats_final<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(ws, n, P, sums, sumsq);
    g_launches++;
  }
  return cudaGetLastError();
}

// ---- symmetric plans: fill the permuted copies inside blocks with repeated
// block indices.  The packed tensor is super-symmetric, so an element whose
// in-block digits are not sorted within a run of equal block indices equals
// the element with those digits sorted (bc/symtensor.py:143-151 reads every
// position through its sorted index the same way); the symmetric moment GEMM
// produces the sorted ones.  One CTA per listed block; reads touch only
// sorted positions, writes only unsorted ones (no hazard).
__global__ void __launch_bounds__(256) k_sym_fill(const int32_t *__restrict__ fill_keys, int64_t nfill,
                                                  const int32_t *__restrict__ keys, const int64_t *__restrict__ offs,
                                                  int m, int b, int64_t n, double *__restrict__ out) {
  for (int64_t w = blockIdx.x; w < nfill; w += gridDim.x) {
    const int32_t k = fill_keys[w];
    const int32_t *key = keys + (int64_t)k * m;
    int e[16], kv[16];
    int size = 1;
#pragma unroll
    for (int q = 0; q < 16; ++q)
      if (q < m) {
        kv[q] = key[q];
        e[q] = (int)(min((int64_t)kv[q] * b, n) - (int64_t)(kv[q] - 1) * b);
        size *= e[q];
      }
    double *blk = out + offs[k];
    for (int i = threadIdx.x; i < size; i += blockDim.x) {
      int d[16];
      int rem = i;
#pragma unroll
      for (int q = 15; q >= 0; --q)
        if (q < m) {
          d[q] = rem % e[q];
          rem /= e[q];
        }
      // insertion sort of the digits within runs of equal block indices
      bool moved = false;
#pragma unroll
      for (int q = 1; q < 16; ++q)
        if (q < m) {
          for (int j = q; j > 0 && kv[j] == kv[j - 1] && d[j] < d[j - 1]; --j) {
            const int tmp = d[j];
            d[j] = d[j - 1];
            d[j - 1] = tmp;
            moved = true;
          }
        }
      if (!moved) continue;
      int lin = 0;
#pragma unroll
      for (int q = 0; q < 16; ++q)
        if (q < m) lin = lin * e[q] + d[q];
      blk[i] = blk[lin];
    }
  }
}

cudaError_t launch_sym_fill(const int32_t *fill_keys, int64_t nfill, const int32_t *keys, const int64_t *offs, int m,
                            int b, int64_t n, double *out, cudaStream_t stream) {
  if (nfill <= 0) return cudaSuccess;
  const int64_t grid = std::min<int64_t>(nfill, 148 * 8);
  k_sym_fill<<<(int)grid, 256, 0, stream>>>(fill_keys, nfill, keys, offs, m, b, n, out);
  return cudaGetLastError();
}

}  // namespace bcg