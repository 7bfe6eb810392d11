// K2 (v2): warp-specialized Khatri-Rao DMMA moment GEMM for sm_100a.
//
// Same mathematics and epilogue mapping as moment.cu (see its header), but the
// three jobs run in separate warps connected by mbarrier rings, so the DMMA
// issue never waits behind a CTA-wide barrier:
//
//   warp 0            TMA warp: 1-D bulk copy (cp.async.bulk) of the sample
//                     chunk X[s:s+KC, :] into an NXS-stage shared ring
//                     (x_full / x_empty barriers; generic copy + zero fill for
//                     a ragged final chunk);
//   warps 1..NPROD    Khatri-Rao builders: per chunk, every A row / B column
//                     factor prod_q X[s+k, col_q] into an NKS-stage ring
//                     (k_full / k_empty); these are the only DMULs;
//   remaining warps   DMMA consumers: mma.sync.m8n8k4.f64 over the KR stage
//                     into a WM x WN register tile, then the packed-address
//                     scatter epilogue (deterministic split-K as in v1).
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"
#include "kr.cuh"
#include "plan.h"

namespace bcg {

namespace {

__device__ __forceinline__ uint32_t s_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_init(uint64_t *b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(b)), "r"(count));
}
__device__ __forceinline__ void bar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_u32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WS_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra.uni WS_DONE;\n"
      "bra.uni WS_WAIT;\n"
      "WS_DONE:\n"
      "}\n" ::"r"(s_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_copy(void *dst, const void *src, uint32_t bytes, uint64_t *b) {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(s_u32(b)), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(s_u32(dst)),
      "l"(src), "r"(bytes), "r"(s_u32(b))
      : "memory");
}
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

}  // namespace

template <int TM, int TN, int WM, int WN, int KC, int NPROD, int NXS, int NKS>
struct WsShape {
  static constexpr int NCONS = (TM / WM) * (TN / WN);
  static constexpr int NWARPS = 1 + NPROD + NCONS;
  static constexpr int NTHREADS = NWARPS * 32;
  static constexpr int LDA = TM + 4;  // == 32 mod 128 bytes: conflict-free fragment loads
  static constexpr int LDB = TN + 4;
  static constexpr int MT = WM / 8, NT = WN / 8;
  static constexpr int JT = TM + TN;  // Khatri-Rao columns built per sample
  static constexpr int NPT = NPROD * 32;
  static constexpr int JPER = (JT + NPT - 1) / NPT;
  static size_t smem(int n) {
    return sizeof(double) * ((size_t)NXS * KC * n + (size_t)NKS * KC * (LDA + LDB)) + 64 * sizeof(uint64_t);
  }
};

template <int TM, int TN, int WM, int WN, int KC, int NPROD, int NXS, int NKS, int M>
__global__ void __launch_bounds__(WsShape<TM, TN, WM, WN, KC, NPROD, NXS, NKS>::NTHREADS, 1)
    k_moment_ws(MomentArgs a) {
  using S = WsShape<TM, TN, WM, WN, KC, NPROD, NXS, NKS>;
  constexpr int H = M / 2, R = M - M / 2;  // compile-time mode counts (0: runtime)
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int n = a.n;
  double *xs = reinterpret_cast<double *>(smem_raw);
  double *kra = xs + (size_t)NXS * KC * n;
  double *krb = kra + (size_t)NKS * KC * S::LDA;
  uint64_t *bars = reinterpret_cast<uint64_t *>(krb + (size_t)NKS * KC * S::LDB);
  uint64_t *x_full = bars, *x_empty = bars + NXS;
  uint64_t *k_full = bars + 2 * NXS, *k_empty = bars + 2 * NXS + NKS;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
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

  if (tid == 0) {
    for (int i = 0; i < NXS; ++i) {
      bar_init(&x_full[i], 1);
      bar_init(&x_empty[i], NPROD);
    }
    for (int i = 0; i < NKS; ++i) {
      bar_init(&k_full[i], NPROD);
      bar_init(&k_empty[i], S::NCONS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA warp
    const uint32_t full_bytes = (uint32_t)(KC * n * sizeof(double));
    for (int c = 0; c < nch; ++c) {
      const int st = c % NXS;
      bar_wait(&x_empty[st], ((c / NXS) & 1) ^ 1);
      double *dst = xs + (size_t)st * KC * n;
      const int64_t s0 = sbeg + (int64_t)c * KC;
      const int rows = (int)(send - s0 < KC ? send - s0 : KC);
      if (rows == KC && a.bulk_ok) {
        if (lane == 0) bulk_copy(dst, a.x + s0 * a.ldx, full_bytes, &x_full[st]);
      } else {
        for (int idx = lane; idx < KC * n; idx += 32) {
          const int rr = idx / n, cc = idx - rr * n;
          dst[idx] = rr < rows ? a.x[(s0 + rr) * a.ldx + cc] : 0.0;
        }
        __syncwarp();
        if (lane == 0) bar_arrive(&x_full[st]);
      }
    }
  } else if (warp <= NPROD) {
    // ------------------------------------------------- Khatri-Rao builders
    const int ptid = tid - 32;
    int cols[S::JPER][8];
    int dsto[S::JPER];   // offset within a KR stage (A or B part), -1 = unused
    bool okj[S::JPER];
    int nq[S::JPER];
#pragma unroll
    for (int u = 0; u < S::JPER; ++u) {
      const int j = ptid + u * S::NPT;
      okj[u] = false;
      dsto[u] = -1;
      nq[u] = 1;
#pragma unroll
      for (int q = 0; q < 8; ++q) cols[u][q] = 0;
      if (j < TM) {
        const int64_t row = (int64_t)tile.row0 + j;
        dsto[u] = j;
        nq[u] = a.h;
        if (row < a.R) {
          okj[u] = true;
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (q < a.h) cols[u][q] = a.rowcols[row * a.h + q];
        }
      } else if (j < S::JT) {
        const int64_t col = (int64_t)tile.col0 + (j - TM);
        dsto[u] = NKS * KC * S::LDA + (j - TM);  // B ring follows the A ring
        nq[u] = a.r;
        if (col < a.C) {
          okj[u] = true;
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (q < a.r) cols[u][q] = a.colcols[col * a.r + q];
        }
      }
    }
    for (int c = 0; c < nch; ++c) {
      const int sx = c % NXS, sk = c % NKS;
      bar_wait(&x_full[sx], (c / NXS) & 1);
      bar_wait(&k_empty[sk], ((c / NKS) & 1) ^ 1);
      const double *xst = xs + (size_t)sx * KC * n;
#pragma unroll
      for (int u = 0; u < S::JPER; ++u) {
        if (dsto[u] < 0) continue;
        const bool isA = dsto[u] < NKS * KC * S::LDA;  // warp-uniform (TM, NPT multiples of 32)
        if (isA) {
          double *dst = kra + dsto[u] + (size_t)sk * KC * S::LDA;
          const double *xr = xst;
#pragma unroll
          for (int k = 0; k < KC; ++k, xr += n) {
            const double p = kr_prod<H>(xr, cols[u], nq[u]);
            dst[k * S::LDA] = okj[u] ? p : 0.0;
          }
        } else {
          double *dst = kra + dsto[u] + (size_t)sk * KC * S::LDB;
          const double *xr = xst;
#pragma unroll
          for (int k = 0; k < KC; ++k, xr += n) {
            const double p = kr_prod<R>(xr, cols[u], nq[u]);
            dst[k * S::LDB] = okj[u] ? p : 0.0;
          }
        }
      }
      __syncwarp();
      if (lane == 0) {
        bar_arrive(&k_full[sk]);
        bar_arrive(&x_empty[sx]);
      }
    }
  } else {
    // ------------------------------------------------------ DMMA consumers
    const int cw = warp - 1 - NPROD;
    const int wm = cw % (TM / WM), wn = cw / (TM / WM);
    const int gid = lane >> 2, tig = lane & 3;
    double acc[S::MT][S::NT][2];
#pragma unroll
    for (int i = 0; i < S::MT; ++i)
#pragma unroll
      for (int j = 0; j < S::NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int c = 0; c < nch; ++c) {
      const int sk = c % NKS;
      bar_wait(&k_full[sk], (c / NKS) & 1);
      const double *ka = kra + (size_t)sk * KC * S::LDA + wm * WM + gid;
      const double *kb = krb + (size_t)sk * KC * S::LDB + wn * WN + gid;
#pragma unroll
      for (int k = 0; k < KC; k += 4) {
        double fa[S::MT], fb[S::NT];
#pragma unroll
        for (int i = 0; i < S::MT; ++i) fa[i] = ka[(k + tig) * S::LDA + 8 * i];
#pragma unroll
        for (int j = 0; j < S::NT; ++j) fb[j] = kb[(k + tig) * S::LDB + 8 * j];
#pragma unroll
        for (int i = 0; i < S::MT; ++i)
#pragma unroll
          for (int j = 0; j < S::NT; ++j) dmma(acc[i][j], fa[i], fb[j]);
      }
      __syncwarp();
      if (lane == 0) bar_arrive(&k_empty[sk]);
    }
    // epilogue: scatter to packed addresses
    double *dst = a.nslices == 1 ? a.out : a.ws + (int64_t)sl_local * a.S;
    const bool accumulate = a.nslices == 1;  // group of one slice: out += partial, in slice order
#pragma unroll
    for (int i = 0; i < S::MT; ++i) {
      const int64_t row = (int64_t)tile.row0 + wm * WM + 8 * i + gid;
      if (row >= a.R) continue;
      const int32_t kb0 = a.row_keybase[row], ro = a.row_olin[row], cs = a.row_cstart[row];
#pragma unroll
      for (int j = 0; j < S::NT; ++j) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t col = (int64_t)tile.col0 + wn * WN + 8 * j + 2 * tig + e;
          if (col >= a.C || col < cs) continue;
          const int32_t key = kb0 + a.col_rank[col];
          if (key < a.kmin_sel || key > a.kmax_sel) continue;
          const int64_t base = a.offs[key];
          if (base < 0) continue;
          const int64_t addr = base + (int64_t)ro * a.col_size[col] + a.col_olin[col];
          if (accumulate)
            dst[addr] += acc[i][j][e];
          else
            dst[addr] = acc[i][j][e];
        }
      }
    }
  }
}

// ----------------------------------------------------------------- variants

#define WS_GO(M, TM, TN, WM, WN, KC, NP, NX, NK) kern = k_moment_ws<TM, TN, WM, WN, KC, NP, NX, NK, M>
#define WS_VARIANT(ID, TM, TN, WM, WN, KC, NP, NX, NK) \
  case ID: {                                            \
    using SH = WsShape<TM, TN, WM, WN, KC, NP, NX, NK>; \
    void (*kern)(MomentArgs) = nullptr;                 \
    BCG_DISPATCH_M(args.h + args.r, WS_GO, TM, TN, WM, WN, KC, NP, NX, NK) \
    const size_t smem = SH::smem(args.n);               \
    if (smem > 227 * 1024) return cudaErrorInvalidValue; \
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    if (e != cudaSuccess) return e;                     \
    if (blocks_per_sm) {                                \
      return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, kern, SH::NTHREADS, smem); \
    }                                                   \
    kern<<<grid, SH::NTHREADS, smem, stream>>>(args);   \
    return cudaGetLastError();                          \
  }

// variant id -> tile shape (must match tile_shape_of below)
cudaError_t launch_moment_ws(const MomentArgs &args, int variant, int grid, cudaStream_t stream,
                             int *blocks_per_sm) {
  switch (variant) {
    WS_VARIANT(1, 128, 64, 32, 32, 16, 3, 3, 3)
    WS_VARIANT(2, 128, 128, 64, 32, 16, 3, 3, 3)
    WS_VARIANT(3, 64, 64, 32, 32, 16, 3, 3, 3)
    WS_VARIANT(4, 128, 128, 32, 32, 16, 3, 3, 2)
    default:
      return cudaErrorInvalidValue;
  }
}

void ws_tile_shape(int variant, int *tm, int *tn) {
  switch (variant) {
    case 1: *tm = 128; *tn = 64; return;
    case 2: *tm = 128; *tn = 128; return;
    case 3: *tm = 64; *tn = 64; return;
    case 4: *tm = 128; *tn = 128; return;
    default: *tm = 64; *tn = 64; return;
  }
}

}  // namespace bcg
