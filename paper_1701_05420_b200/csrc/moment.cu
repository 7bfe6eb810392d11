// K2: order-m packed moment as a Khatri-Rao-staged FP64 DMMA GEMM (sm_100a).
//
// Reference semantics: bc/_core.pyx:60-148 (raw product sums accumulated into
// the packed buffer).  Formulation: bc/_engines.py:141-208 (gram engine) --
// every stored block (L, R) is the sub-matrix W_L^T W_R of the Gram matrix of
// Khatri-Rao product columns, here restricted to the useful staircase
// {row group v = L[-1], col R with R[0] >= v} so nothing outside S_m is formed
// except ragged tile edges.
//
// Input: the TRANSPOSED data xt (n rows x ldt, one contiguous row per
// variable -- the layout the reference's own kernel takes, bc/_engines.py:95),
// zero-padded to a multiple of 16 samples.
//
// Per CTA (TM x TN output tile, 4 warps):
//   1. a sample chunk xt[:, s:s+16] is staged into shared memory by ONE 2-D TMA
//      tensor copy (cp.async.bulk.tensor, box 16 samples x n variables, SASS
//      UTMALDG) with 128-byte swizzle (8 consecutive rows at the same sample
//      pair hit 8 distinct 16-byte bank groups), double buffered, on an
//      mbarrier;
//   2. the chunk's Khatri-Rao factors A[i][k] = prod_q X[s+k, rowcols[i][q]]
//      and B[j][k] are built in shared memory (never in HBM), two samples per
//      LDS.128 / DMUL pair / STS.128, at compile-time offsets;
//   3. warps run mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4) over the chunk into FP64
//      register tiles; the loop is software-pipelined (the factors of chunk c+1
//      are built while chunk c's DMMAs issue, one CTA barrier per chunk);
//   4. the epilogue scatters each accumulator to its packed address
//      koff[keybase[row] + rank[col]] + olin[row] * size[col] + olin[col],
//      either accumulating into `out` (one K-slice per launch) or writing a
//      per-slice partial that k_reduce_slices adds in slice order
//      (deterministic split-K, no float atomics).  Slices have a fixed length
//      (kSliceLen samples), so every element's summation order depends on t
//      only -- not on the plan, tile shape, key range or launch grouping.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "kernels.h"
#include "kr.cuh"
#include "plan.h"

#ifndef BCG_MOMENT_PART
#error "moment.cu is compiled once per BCG_MOMENT_PART (0..8), see _build.py"
#endif

namespace bcg {

constexpr int kThreads = 128;
// CTA threads of a tile shape: 4 warps, or 8 for the 8192-element tiles
// (128 x 64, 64 x 128: a 32 x 32 warp tile each, half the Khatri-Rao build
// per FMA of one dimension)
__host__ __device__ constexpr int moment_threads(int tm, int tn) { return tm * tn >= 8192 ? 256 : 128; }

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
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void mbar_expect(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

// CTA tile TM x TN, 4 warps in a WGM x WGN grid (warp tile WM x WN of 8x8
// DMMA sub-tiles).  Factor storage [row][k], 16 doubles per row, the 16-byte
// sample-pair chunks of row r XOR-swizzled by s(r) = 2 (r & 3) + ((r >> 2) & 1)
// (kr_swizzle returns 2 s(r), the swizzle of the double index):
//   * a paired STS.128 of 8 consecutive rows (a quarter warp, one sample pair)
//     hits 8 distinct chunks;
//   * an m8n8k4 fragment load (half warp: rows gid = 0..3 or 4..7, samples
//     k0 + tig) hits 16 distinct doubles, since s(r) >> 1 = r & 3.
// (The previous (r & 3) << 2 left the stores 2-way conflicted: 17% of the
// kernel's shared-memory wavefronts at cfg4, profiles/r02_moment_cfg4_ncu.txt.)
__device__ __forceinline__ int kr_swizzle(int row) { return ((row & 3) << 2) | ((row >> 1) & 2); }

template <int KC, int TM, int TN>
struct V1Shape {
  static constexpr int NTH = moment_threads(TM, TN);
  static constexpr int NW = NTH / 32;
  static constexpr int WGN = NW == 8 ? TN / 32 : (TN >= 4 * TM ? 4 : (TN >= TM ? 2 : 1));
  static constexpr int WGM = NW / WGN;
  static constexpr int WM = TM / WGM, WN = TN / WGN;
  static constexpr int MT = WM / 8, NT = WN / 8;
  static constexpr int LDK = KC;       // factor row stride (doubles), swizzled
  static_assert(KC == 16, "the TMA box is one 128-byte swizzle span of samples");
  static constexpr int PA = NTH / TM, PB = NTH / TN;  // threads per factor row
  static constexpr int NPAIR = KC / 2;                // sample pairs per chunk
  static_assert(WGM * WGN == NW, "warp grid");
  static_assert(WM % 8 == 0 && WN % 8 == 0, "warp tile must be a multiple of 8");
  static_assert(NTH % TM == 0 && NTH % TN == 0, "TM, TN must divide the CTA threads");
  static_assert(NPAIR % PA == 0 && NPAIR % PB == 0, "sample pairs must split evenly");
};

// samples (2j, 2j+1) of staged row r: 128-byte swizzle, 16-byte chunk j of
// row r lives at chunk j ^ (r & 7)
__device__ __forceinline__ double2 xs_pair(const double *row, int sw, int j) {
  return *reinterpret_cast<const double2 *>(row + 2 * (j ^ sw));
}

template <int NQ>
__device__ __forceinline__ double2 kr_pair(const double *const (&row)[8], const int (&sw)[8], int nq, int j) {
  double2 p = xs_pair(row[0], sw[0], j);
  if constexpr (NQ > 0) {
#pragma unroll
    for (int q = 1; q < NQ; ++q) {
      const double2 v = xs_pair(row[q], sw[q], j);
#ifdef BCG_EXP_NODMUL
      // timing experiment only (results are wrong): the same loads and stores, no FP64 multiply
      p.x = __longlong_as_double(__double_as_longlong(p.x) ^ __double_as_longlong(v.x));
      p.y = __longlong_as_double(__double_as_longlong(p.y) ^ __double_as_longlong(v.y));
#else
      p.x *= v.x;
      p.y *= v.y;
#endif
    }
  } else {
#pragma unroll
    for (int q = 1; q < 8; ++q)
      if (q < nq) {
        const double2 v = xs_pair(row[q], sw[q], j);
        p.x *= v.x;
        p.y *= v.y;
      }
  }
  return p;
}

// H, R: compile-time row / column mode counts (0: the runtime a.h / a.r)
template <int KC, int H, int R, int TM, int TN>
__global__ void __launch_bounds__(moment_threads(TM, TN)) k_moment_dmma(const __grid_constant__ CUtensorMap tmap,
                                                                        MomentArgs a) {
  using SH = V1Shape<KC, TM, TN>;
  constexpr int LDX = KC;                  // staged row: 16 doubles = one 128-byte swizzle span
  constexpr int LDK = SH::LDK, MT = SH::MT, NT = SH::NT;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int n = a.n;
  const int xstaged = xstaged_rows(n);                 // TMA-staged variable rows (>= n)
  const int xrows = (xstaged + 7) / 8 * 8;             // 1024-byte stages
  double *xs = reinterpret_cast<double *>(smem_raw);   // [2][xrows][16], swizzled
  double *kra = xs + 2 * xrows * LDX;                  // [2][TM][LDK]
  double *krb = kra + 2 * TM * LDK;                    // [2][TN][LDK]
  uint64_t *bar = reinterpret_cast<uint64_t *>(krb + 2 * TN * LDK);

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
  const int nch = (int)((send - sbeg + KC - 1) / KC);  // xt is zero-padded past t

  // ---- per-thread Khatri-Rao assignment: a fixed factor row (A) and column
  // (B), an interleaved set of sample pairs.  Rows past R / C keep column 0:
  // their products feed only accumulators the epilogue discards. ----
  const int ia = tid % TM, pa0 = tid / TM;
  const int ib = tid % TN, pb0 = tid / TN;
  int colA[8], colB[8];
  {
    const int64_t grow = (int64_t)tile.row0 + ia;
    const int64_t gcol = (int64_t)tile.col0 + ib;
    const bool okA = grow < a.R, okB = gcol < a.C;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      colA[q] = (okA && q < a.h) ? a.rowcols[grow * a.h + q] : 0;
      colB[q] = (okB && q < a.r) ? a.colcols[gcol * a.r + q] : 0;
      BCG_CHECK(colA[q] >= 0 && colA[q] < xstaged, "colA", colA[q]);
      BCG_CHECK(colB[q] >= 0 && colB[q] < xstaged, "colB", colB[q]);
    }
  }

  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // thread 0 stages chunk c: one 2-D tensor copy per 256 variables
  auto issue = [&](int c) {
    if (tid == 0) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      // every box transfers its full height (rows past n are zero-filled)
      mbar_expect(&bar[c & 1], (uint32_t)(xstaged * KC * sizeof(double)));
      double *dst = xs + (c & 1) * xrows * LDX;
      const int s0 = (int)(sbeg + (int64_t)c * KC);
      const int bh = xbox_rows(n);
      for (int v0 = 0; v0 < xstaged; v0 += bh) tma_load_2d(dst + v0 * LDX, &tmap, s0, v0, &bar[c & 1]);
    }
  };

  const int warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int wm = warp % SH::WGM, wn = warp / SH::WGM;
  // acc[i][j][e] = C[8i + gid][8j + 2 tig + e] (m8n8k4 accumulator fragments)
  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  auto build_a = [&](int c) {  // row factors of chunk c -> kra[c & 1] (waits for the chunk)
    mbar_wait(&bar[c & 1], (uint32_t)((c >> 1) & 1));
#ifdef BCG_EXP_NOBUILD
    return;  // timing experiment only (results are wrong): the kernel without the Khatri-Rao build
#endif
    const double *xst = xs + (c & 1) * xrows * LDX;
    {
      const double *ra[8];
      int sa[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        ra[q] = xst + colA[q] * LDX;
        sa[q] = colA[q] & 7;
      }
      double *wa = kra + (c & 1) * TM * LDK + ia * LDK;
      const int swa = kr_swizzle(ia);
#pragma unroll
      for (int i = 0; i < SH::NPAIR / SH::PA; ++i) {
        const int j = pa0 + SH::PA * i;
        const double2 p = kr_pair<H>(ra, sa, a.h, j);
        *reinterpret_cast<double2 *>(wa + ((2 * j) ^ swa)) = p;
      }
    }
  };
  auto build_b = [&](int c) {  // column factors of chunk c -> krb[c & 1]
#ifdef BCG_EXP_NOBUILD
    return;
#endif
    const double *xst = xs + (c & 1) * xrows * LDX;
    {
      const double *rb[8];
      int sb[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        rb[q] = xst + colB[q] * LDX;
        sb[q] = colB[q] & 7;
      }
      double *wb = krb + (c & 1) * TN * LDK + ib * LDK;
      const int swb = kr_swizzle(ib);
#pragma unroll
      for (int i = 0; i < SH::NPAIR / SH::PB; ++i) {
        const int j = pb0 + SH::PB * i;
        const double2 p = kr_pair<R>(rb, sb, a.r, j);
        *reinterpret_cast<double2 *>(wb + ((2 * j) ^ swb)) = p;
      }
    }
  };
  auto build = [&](int c) {  // Khatri-Rao factors of chunk c -> kra/krb[c & 1]
    build_a(c);
    build_b(c);
  };

  if (nch > 0) {
    issue(0);
    if (nch > 1) issue(1);
    build(0);
    __syncthreads();  // KR[0] complete, xs[0] free
    if (nch > 2) issue(2);
  }
  for (int c = 0; c < nch; ++c) {
    // ---- DMMA over chunk c ----
    // fragment rows = gid (mod 8 after the 8-row and warp offsets), sample
    // k + tig: double index (k + tig) ^ kr_swizzle(gid)
    const int swf = kr_swizzle(gid);
    const double *ka = kra + (c & 1) * TM * LDK + (wm * SH::WM + gid) * LDK;
    const double *kb = krb + (c & 1) * TN * LDK + (wn * SH::WN + gid) * LDK;
    auto ksteps = [&](int k0, int k1) {
#pragma unroll
      for (int k = k0; k < k1; k += 4) {
        double fa[MT], fb[NT];
        const int ks = (k + tig) ^ swf;
#pragma unroll
        for (int i = 0; i < MT; ++i) fa[i] = ka[8 * i * LDK + ks];
#pragma unroll
        for (int j = 0; j < NT; ++j) fb[j] = kb[8 * j * LDK + ks];
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int j = 0; j < NT; ++j) dmma884(acc[i][j], fa[i], fb[j]);
      }
    };
    if constexpr (H >= 3 && R >= 3) {
      // three-mode factors (m = 6): the column factors of chunk c+1 are built
      // between the two halves of chunk c's DMMAs (+0.6 points of DMMA peak at
      // cfg4; -0.5 at cfg2's two-mode factors, which keep one build phase;
      // profiles/r01_moment_schedule_experiments.log (5))
      if (c + 1 < nch) build_a(c + 1);
      ksteps(0, KC / 2);
      if (c + 1 < nch) build_b(c + 1);
      ksteps(KC / 2, KC);
    } else {
      if (c + 1 < nch) build(c + 1);
      ksteps(0, KC);
    }
    __syncthreads();  // KR[c+1] complete, KR[c] and xs[(c+1) & 1] free
    if (c + 3 < nch) issue(c + 3);
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
        const int64_t addr = base + (int64_t)ro * a.col_size[col] + a.col_olin[col];
        BCG_CHECK(addr >= 0 && addr < a.S, "epilogue address", addr);
        if (accumulate)
          dst[addr] += acc[i][j][e];
        else
          dst[addr] = acc[i][j][e];
      }
    }
  }
}

#if BCG_MOMENT_PART == 0
// ---- part 0: shape-independent host code, the split-K reduce, dispatch ----
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
  const size_t xrows = (size_t)(xstaged_rows(n) + 7) / 8 * 8;
  return sizeof(double) * (2 * xrows * KC + 2 * (size_t)(tm + tn) * KC) + 2 * sizeof(uint64_t) +
         1024;  // + alignment slack for the 1024-byte swizzle atoms
}

int pick_kc(int n) {  // 16-sample chunks (one 128-byte swizzle span) while they fit
  return moment_smem_bytes(16, n, 64, 64) <= 227 * 1024 ? 16 : 0;
}

// tile shapes: 64x64 for every KC / order; the thin / small shapes
// (staircase-friendly, chosen per plan by the tile model) for KC = 16 and
// orders 2..8.
bool v1_shape_supported(int KC, int m, int tm, int tn) {
  if (KC != 16) return false;
  if (tm == 64 && tn == 64) return true;
  if (m < 2 || m > 8) return false;
  return (tm == 16 && tn == 128) || (tm == 128 && tn == 16) || (tm == 32 && tn == 64) ||
         (tm == 64 && tn == 32) || (tm == 32 && tn == 32) || (tm == 128 && tn == 64) || (tm == 64 && tn == 128);
}

#define BCG_SHAPE_DECL(TMV, TNV) \
  cudaError_t launch_moment_##TMV##x##TNV(const MomentArgs &args, int grid, cudaStream_t stream, bool generic);
BCG_SHAPE_DECL(64, 64)
BCG_SHAPE_DECL(16, 128)
BCG_SHAPE_DECL(128, 16)
BCG_SHAPE_DECL(32, 64)
BCG_SHAPE_DECL(64, 32)
BCG_SHAPE_DECL(32, 32)
BCG_SHAPE_DECL(128, 64)
BCG_SHAPE_DECL(64, 128)
#undef BCG_SHAPE_DECL

cudaError_t launch_moment(const MomentArgs &args, int KC, int grid, cudaStream_t stream, int tm, int tn) {
  static const bool generic = getenv("BCG_FORCE_GENERIC_M") != nullptr;  // debug knob
  const int h = args.h, r = args.r;
  if (KC != 16 || h < 1 || r < 1 || h > 8 || r > 8) return cudaErrorInvalidValue;
  if (!v1_shape_supported(KC, h + r, tm, tn)) return cudaErrorInvalidValue;
#define GO(TMV, TNV) \
  if (tm == TMV && tn == TNV) return launch_moment_##TMV##x##TNV(args, grid, stream, generic);
  GO(64, 64) GO(16, 128) GO(128, 16) GO(32, 64) GO(64, 32) GO(32, 32) GO(128, 64) GO(64, 128)
#undef GO
  return cudaErrorInvalidValue;
}

cudaError_t launch_reduce_slices(const double *ws, int nslices, int64_t S, int64_t lo, int64_t hi,
                                 double *out, cudaStream_t stream) {
  if (hi <= lo) return cudaSuccess;
  int64_t blocks = (hi - lo + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_reduce_slices<<<(int)blocks, 256, 0, stream>>>(ws, nslices, S, lo, hi, out);
  return cudaGetLastError();
}

#else
// ---- parts 1..6: the kernel instantiations of one CTA tile shape each
// (separate translation units so nvcc compiles them in parallel) ----
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D map over xt (inner: padded samples, outer: variables), box 16 x min(n, 256),
// 128-byte swizzle
static cudaError_t make_xt_map(const MomentArgs &a, CUtensorMap *map) {
  auto enc = tensor_map_encoder();
  if (!enc) return cudaErrorNotSupported;
  cuuint64_t dims[2] = {(cuuint64_t)a.ldx, (cuuint64_t)a.n};
  cuuint64_t strides[1] = {(cuuint64_t)a.ldx * sizeof(double)};
  cuuint32_t box[2] = {16, (cuuint32_t)xbox_rows(a.n)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(a.x), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int KC, int H, int R, int TM, int TN>
static cudaError_t go_v1(const MomentArgs &args, int grid, cudaStream_t stream) {
  const size_t smem = moment_smem_bytes(KC, args.n, TM, TN);
  auto kern = k_moment_dmma<KC, H, R, TM, TN>;
  CUtensorMap map;
  cudaError_t e = make_xt_map(args, &map);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, moment_threads(TM, TN), smem, stream>>>(map, args);
  return cudaGetLastError();
}

// (h | r) splits with a compiled specialization: the balanced split of every
// order 2..8 and, for odd orders, its mirror (the second GEMM of a hybrid plan);
// other splits (orders 9..16) take the runtime-mode-count kernel (64 x 64)
#define BCG_SHAPE_DEF(TMV, TNV)                                                                        \
  cudaError_t launch_moment_##TMV##x##TNV(const MomentArgs &args, int grid, cudaStream_t stream,        \
                                          bool generic) {                                              \
    const int h = args.h, r = args.r;                                                                  \
    if (!generic) {                                                                                    \
      BCG_SPLIT(1, 1) BCG_SPLIT(1, 2) BCG_SPLIT(2, 1) BCG_SPLIT(2, 2) BCG_SPLIT(2, 3) BCG_SPLIT(3, 2) \
      BCG_SPLIT(3, 3) BCG_SPLIT(3, 4) BCG_SPLIT(4, 3) BCG_SPLIT(4, 4)                                  \
    }                                                                                                  \
    if constexpr (TMV == 64 && TNV == 64) return go_v1<16, 0, 0, TMV, TNV>(args, grid, stream);      \
    else                                                                                               \
    return cudaErrorInvalidValue;                                                                      \
  }
#define BCG_SPLIT(HV, RV) \
  if (h == HV && r == RV) return go_v1<16, HV, RV, TMV_, TNV_>(args, grid, stream);

#if BCG_MOMENT_PART == 1
#define TMV_ 64
#define TNV_ 64
#elif BCG_MOMENT_PART == 2
#define TMV_ 16
#define TNV_ 128
#elif BCG_MOMENT_PART == 3
#define TMV_ 128
#define TNV_ 16
#elif BCG_MOMENT_PART == 4
#define TMV_ 32
#define TNV_ 64
#elif BCG_MOMENT_PART == 5
#define TMV_ 64
#define TNV_ 32
#elif BCG_MOMENT_PART == 6
#define TMV_ 32
#define TNV_ 32
#elif BCG_MOMENT_PART == 7
#define TMV_ 128
#define TNV_ 64
#elif BCG_MOMENT_PART == 8
#define TMV_ 64
#define TNV_ 128
#endif
#define BCG_DEF_EXPAND(A, B) BCG_SHAPE_DEF(A, B)
BCG_DEF_EXPAND(TMV_, TNV_)
#endif  // BCG_MOMENT_PART

}  // namespace bcg
