// K2: order-m packed moment as a Khatri-Rao-staged FP64 DMMA GEMM (sm_100a).
//
// Reference semantics: bc/_core.pyx:60-148 (raw product sums accumulated into
// the packed buffer).  Formulation: bc/_engines.py:141-208 (gram engine) --
// every stored block (L, R) is the sub-matrix W_L^T W_R of the Gram matrix of
// Khatri-Rao product columns, here restricted to the useful staircase
// {row group v = L[-1], col R with R[0] >= v} so nothing outside S_m is formed
// except ragged tile edges.
//
// Per CTA (64 x 64 output tile, 4 warps of 32 x 32):
//   1. a contiguous sample chunk X[s:s+KC, :] is staged into shared memory by
//      a 1-D TMA bulk copy (cp.async.bulk, mbarrier complete_tx), double
//      buffered;
//   2. the chunk's Khatri-Rao factors  A[k][i] = prod_q X[s+k, rowcols[i][q]]
//      and B[k][j] = prod_q X[s+k, colcols[j][q]] are built in shared memory
//      (never in HBM), double buffered;
//   3. warps run mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4) over the chunk, FP64
//      accumulators in registers;
//   4. the epilogue scatters each accumulator to its packed address
//      offs[keybase[row] + rank[col]] + olin[row] * size[col] + olin[col],
//      either accumulating into `out` (one K-slice) or writing a per-slice
//      partial that k_reduce_slices adds in slice order (deterministic split-K,
//      no float atomics).  Slices have a fixed length (kSliceLen samples), so
//      every element's summation order depends on t only -- not on the plan,
//      tile shape, key range or launch grouping: moments from different plans
//      (block-split, kernel variants) agree bitwise.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "kernels.h"
#include "kr.cuh"
#include "plan.h"

namespace bcg {

constexpr int kPad = 4;  // row stride (TM + 4) doubles == 32 mod 128 bytes: the 4 k-rows of an m8n8k4 fragment load hit 4 distinct bank quadrants (conflict-free)
constexpr int kThreads = 128;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra.uni DONE;\n"
      "bra.uni LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity));
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// CTA tile TM x TN, 4 warps in a WGM x WGN grid (warp tile WM x WN of 8x8
// DMMA sub-tiles).  Khatri-Rao work split: TM rows x KC samples of A and
// TN columns x KC samples of B over 128 threads, each thread a fixed row
// (column) and an interleaved set of samples, so its X column indices stay in
// registers.
template <int TM, int TN>
struct V1Shape {
  static constexpr int WGN = TN >= 4 * TM ? 4 : (TN >= TM ? 2 : 1);
  static constexpr int WGM = 4 / WGN;
  static constexpr int WM = TM / WGM, WN = TN / WGN;
  static constexpr int MT = WM / 8, NT = WN / 8;
  static constexpr int LDA = TM + kPad, LDB = TN + kPad;
  static_assert(WM % 8 == 0 && WN % 8 == 0, "warp tile must be a multiple of 8");
  static_assert(kThreads % TM == 0 && kThreads % TN == 0, "TM, TN must divide 128");
};

template <int KC, int M, bool ONES, int TM, int TN>
__global__ void __launch_bounds__(kThreads) k_moment_dmma(MomentArgs a) {
  using SH = V1Shape<TM, TN>;
  constexpr int H = M / 2, R = M - M / 2;  // compile-time mode counts (0: runtime)
  constexpr int LDA = SH::LDA, LDB = SH::LDB, MT = SH::MT, NT = SH::NT;
  constexpr int PA = kThreads / TM, PB = kThreads / TN;  // sample phases per row / col
  static_assert(KC % PA == 0 && KC % PB == 0, "KC must be a multiple of the sample phases");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int n = a.n;
  double *xs = reinterpret_cast<double *>(smem_raw);   // [2][KC*n]
  double *kra = xs + 2 * KC * n;                       // [2][KC][LDA]
  double *krb = kra + 2 * KC * LDA;                    // [2][KC][LDB]
  uint64_t *bar = reinterpret_cast<uint64_t *>(krb + 2 * KC * LDB);

  const int tid = threadIdx.x;
  const int unit = blockIdx.x;
  const int sl_local = unit / a.ntiles;  // slice within this launch's group
  const int tile_id = unit - sl_local * a.ntiles;
  const int slice = a.slice0 + sl_local;
  if (a.kmin_sel > 0 || a.kmax_sel < INT32_MAX) {
    if (a.tile_kmax[tile_id] < a.kmin_sel || a.tile_kmin[tile_id] > a.kmax_sel) return;
  }
  const Tile tile = a.tiles[tile_id];
  const int64_t sbeg = (int64_t)slice * a.slice_len;
  const int64_t send = min(a.t, sbeg + a.slice_len);
  const int64_t slen = send - sbeg;
  const int nch = (int)((slen + KC - 1) / KC);

  // ---- per-thread Khatri-Rao assignment ----
  const int ia = tid % TM, pa0 = tid / TM;  // A row, first sample phase (step PA)
  const int ib = tid % TN, pb0 = tid / TN;  // B col, first sample phase (step PB)
  int colA[8], colB[8];
  const int64_t grow = (int64_t)tile.row0 + ia;
  const int64_t gcol = (int64_t)tile.col0 + ib;
  const bool okA = grow < a.R, okB = gcol < a.C;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    colA[q] = (okA && q < a.h) ? a.rowcols[grow * a.h + q] : 0;
    colB[q] = (okB && q < a.r) ? a.colcols[gcol * a.r + q] : 0;
  }

  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  const uint32_t full_bytes = (uint32_t)(KC * n * sizeof(double));
  auto chunk_full = [&](int c) { return (int64_t)(c + 1) * KC <= slen && a.bulk_ok; };
  auto issue = [&](int c) {
    const double *src = a.x + (sbeg + (int64_t)c * KC) * a.ldx;
    bulk_g2s(xs + (c & 1) * KC * n, src, full_bytes, &bar[c & 1]);
  };

  const int warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int wm = warp % SH::WGM, wn = warp / SH::WGM;
  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // Software pipeline, one CTA barrier per chunk: while the warps issue the
  // DMMAs of chunk c they also build the Khatri-Rao factors of chunk c+1 into
  // the other KR buffer; the TMA copy of chunk c+2 is in flight meanwhile.
  //   stage(x) = x & 1 for both the X ring and the KR double buffer.
  auto load_x = [&](int c) {  // make chunk c's samples resident in xs[c & 1]
    double *xst = xs + (c & 1) * KC * n;
    if (chunk_full(c)) {
      mbar_wait(&bar[c & 1], (uint32_t)((c >> 1) & 1));
    } else {
      // ragged / strided chunk: plain loads, zero-filled past the slice end
      const int64_t s0 = sbeg + (int64_t)c * KC;
      const int rows = (int)(send - s0 < KC ? send - s0 : KC);
      for (int idx = tid; idx < KC * n; idx += kThreads) {
        const int rr = idx / n, cc = idx - rr * n;
        xst[idx] = rr < rows ? a.x[(s0 + rr) * a.ldx + cc] : 0.0;
      }
      __syncthreads();
    }
  };
  auto build = [&](int c) {  // Khatri-Rao factors of chunk c -> kra/krb[c & 1]
    const double *xst = xs + (c & 1) * KC * n;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      BCG_CHECK(colA[q] >= (ONES ? -1 : 0) && colA[q] < n, "colA", colA[q]);
      BCG_CHECK(colB[q] >= (ONES ? -1 : 0) && colB[q] < n, "colB", colB[q]);
    }
    {
      double *wa = kra + (c & 1) * KC * LDA + pa0 * LDA + ia;
      const double *xr = xst + pa0 * n;
#pragma unroll
      for (int k = 0; k < KC / PA; ++k) {
        const double p = kr_prod<H, ONES>(xr, colA, a.h);
        wa[k * PA * LDA] = okA ? p : 0.0;
        xr += PA * n;
      }
    }
    {
      double *wb = krb + (c & 1) * KC * LDB + pb0 * LDB + ib;
      const double *xr = xst + pb0 * n;
#pragma unroll
      for (int k = 0; k < KC / PB; ++k) {
        const double p = kr_prod<R, ONES>(xr, colB, a.r);
        wb[k * PB * LDB] = okB ? p : 0.0;
        xr += PB * n;
      }
    }
  };

  if (nch > 0) {
    if (tid == 0) {
      if (chunk_full(0)) issue(0);
      if (nch > 1 && chunk_full(1)) issue(1);
    }
    load_x(0);
    build(0);
    __syncthreads();
    if (tid == 0 && nch > 2 && chunk_full(2)) issue(2);
  }
  for (int c = 0; c < nch; ++c) {
    if (c + 1 < nch) {
      load_x(c + 1);
      build(c + 1);
    }
    // ---- DMMA over chunk c ----
    const double *ka = kra + (c & 1) * KC * LDA;
    const double *kb = krb + (c & 1) * KC * LDB;
#pragma unroll
    for (int k = 0; k < KC; k += 4) {
      double fa[MT], fb[NT];
      const double *pa = ka + (k + tig) * LDA + wm * SH::WM + gid;
      const double *pb = kb + (k + tig) * LDB + wn * SH::WN + gid;
#pragma unroll
      for (int i = 0; i < MT; ++i) fa[i] = pa[8 * i];
#pragma unroll
      for (int j = 0; j < NT; ++j) fb[j] = pb[8 * j];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma884(acc[i][j], fa[i], fb[j]);
    }
    __syncthreads();  // KR[c+1] complete, KR[c] and xs[(c+1) & 1] free
    if (tid == 0 && c + 3 < nch && chunk_full(c + 3)) issue(c + 3);
  }

  // ---- epilogue: scatter to packed addresses ----
  double *dst = a.nslices == 1 ? a.out : a.ws + (int64_t)sl_local * a.S;
  const bool accumulate = a.nslices == 1;  // group of one slice: out += partial, in slice order
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const int64_t row = (int64_t)tile.row0 + wm * SH::WM + 8 * i + gid;
    if (row >= a.R) continue;
    const int32_t kb0 = a.row_keybase[row], ro = a.row_olin[row], cs = a.row_cstart[row];
#pragma unroll
    for (int j = 0; j < NT; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t col = (int64_t)tile.col0 + wn * SH::WN + 8 * j + 2 * tig + e;
        if (col >= a.C || col < cs) continue;
        const int32_t key = kb0 + a.col_rank[col];
        if (key < a.kmin_sel || key > a.kmax_sel) continue;
        const int64_t base = a.offs[key];  // output offset of the key's block
        if (base < 0) continue;            // fused plan: orders 0 / 1 are not produced
        const int64_t addr = base + (int64_t)ro * a.col_size[col] + a.col_olin[col];
        BCG_CHECK(addr >= 0 && addr < a.S, "epilogue address", addr);
        BCG_CHECK(key >= 0, "key", key);
        if (accumulate)
          dst[addr] += acc[i][j][e];
        else
          dst[addr] = acc[i][j][e];
      }
    }
  }
}

// out[i] = ((out[i] + ws[0][i]) + ws[1][i]) + ...  for i in [lo, hi): the
// slices of one group added sequentially, so the association of the whole
// split-K sum is the same for any grouping of the slices.
__global__ void k_reduce_slices(const double *__restrict__ ws, int nslices, int64_t S, int64_t lo,
                                int64_t hi, double *__restrict__ out) {
  for (int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hi;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = out[i];
    for (int k = 0; k < nslices; ++k) v += ws[k * S + i];
    out[i] = v;
  }
}

size_t moment_smem_bytes(int KC, int n, int tm, int tn) {
  return sizeof(double) * (2 * (size_t)KC * n + 2 * (size_t)KC * (tm + kPad) + 2 * (size_t)KC * (tn + kPad)) +
         2 * sizeof(uint64_t);
}

int pick_kc(int n) {  // sample-chunk length for the 64x64 tile
  // keep the double-buffered sample stage <= 96 KB so >= 2 CTAs fit per SM
  if (2 * 16 * (size_t)n * 8 <= 96 * 1024) return 16;
  if (2 * 8 * (size_t)n * 8 <= 96 * 1024) return 8;
  if (2 * 4 * (size_t)n * 8 <= 160 * 1024) return 4;
  return 0;
}

template <int KC, int M, int TM, int TN>
static cudaError_t go_v1(const MomentArgs &args, int grid, cudaStream_t stream) {
  const size_t smem = moment_smem_bytes(KC, args.n, TM, TN);
  auto kern = args.ones ? k_moment_dmma<KC, M, true, TM, TN> : k_moment_dmma<KC, M, false, TM, TN>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, kThreads, smem, stream>>>(args);
  return cudaGetLastError();
}

// v1 tile shapes: 64x64 for every KC / order; the thin / small shapes
// (staircase-friendly, chosen per plan by the tile model) for KC = 16 and
// orders 2..8.
bool v1_shape_supported(int KC, int m, int tm, int tn) {
  if (tm == 64 && tn == 64) return true;
  if (KC != 16 || m < 2 || m > 8) return false;
  return (tm == 16 && tn == 128) || (tm == 128 && tn == 16) || (tm == 32 && tn == 64) ||
         (tm == 64 && tn == 32) || (tm == 32 && tn == 32);
}

cudaError_t launch_moment(const MomentArgs &args, int KC, int grid, cudaStream_t stream, int tm, int tn) {
  static const bool generic = getenv("BCG_FORCE_GENERIC_M") != nullptr;  // debug knob
  const int m = generic ? 0 : args.h + args.r;
  cudaError_t e = cudaErrorInvalidValue;
  if (!(tm == 64 && tn == 64)) {
    if (!v1_shape_supported(KC, m, tm, tn)) return cudaErrorInvalidValue;
#define GOS(M, TMV, TNV) e = go_v1<16, M, TMV, TNV>(args, grid, stream)
#define SHAPE(TMV, TNV)                                   \
  if (tm == TMV && tn == TNV) {                           \
    switch (m) {                                          \
      case 2: GOS(2, TMV, TNV); break;                    \
      case 3: GOS(3, TMV, TNV); break;                    \
      case 4: GOS(4, TMV, TNV); break;                    \
      case 5: GOS(5, TMV, TNV); break;                    \
      case 6: GOS(6, TMV, TNV); break;                    \
      case 7: GOS(7, TMV, TNV); break;                    \
      case 8: GOS(8, TMV, TNV); break;                    \
      default: break;                                     \
    }                                                     \
    return e;                                             \
  }
    SHAPE(16, 128)
    SHAPE(128, 16)
    SHAPE(32, 64)
    SHAPE(64, 32)
    SHAPE(32, 32)
#undef SHAPE
#undef GOS
    return e;
  }
#define GO16(M, ...) e = go_v1<16, M, 64, 64>(args, grid, stream)
#define GO8(M, ...) e = go_v1<8, M, 64, 64>(args, grid, stream)
#define GO4(M, ...) e = go_v1<4, M, 64, 64>(args, grid, stream)
  switch (KC) {
    case 16: BCG_DISPATCH_M(m, GO16, 0) break;
    case 8: BCG_DISPATCH_M(m, GO8, 0) break;
    case 4: BCG_DISPATCH_M(m, GO4, 0) break;
    default: break;
  }
#undef GO16
#undef GO8
#undef GO4
  return e;
}

cudaError_t launch_reduce_slices(const double *ws, int nslices, int64_t S, int64_t lo, int64_t hi,
                                 double *out, cudaStream_t stream) {
  if (hi <= lo) return cudaSuccess;
  int64_t blocks = (hi - lo + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_reduce_slices<<<(int)blocks, 256, 0, stream>>>(ws, nslices, S, lo, hi, out);
  return cudaGetLastError();
}

}  // namespace bcg
