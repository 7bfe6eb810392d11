// K3 (v2): cumulant recursion at memory rate, for full blocks (all edges = b).
//
// Uses the moment-cumulant relation of centered data expanded by the part
// that contains mode 1 (PAPER.md:650-666 restated by subsets):
//
//   M(1..m) = sum_{S containing 1} C(S) * M(rest),   M(empty) = 1, M(single) = 0
//   =>  C_m = M_m - sum_{S containing 1, 2 <= |S| <= m-2} C_|S|[key|S] * M_{m-|S|}[key|rest]
//
// which is algebraically the reference's partition sum (bc/cumulants.py:53-136:
// grouping the partitions by the part holding mode 1 turns the sum over the
// other parts into the central moment of the complement).  m = 6: 25 products
// instead of 40 partitions / 55 multiplications.  M_2 = C_2 and M_3 = C_3; the
// central moments M_4.. of the complement are kept by the caller.
//
// Every sub-key of a sorted key is sorted, so each factor is an element of a
// stored lower-order block (bc/cumulants.py:9-12); the host precomputes the
// element offset of each term's two factor blocks per output block.
//
// Register blocking: a thread owns one trailing index of the output block and
// the B^(m-CT) elements sharing it in registers.  The term list, the factor
// strides and the row offsets are compile-time (template on m and B), so every
// factor access is a per-thread base plus an immediate offset; lanes cover
// consecutive elements, so M_m is read and C_m written coalesced (HBM-bound:
// 16 bytes per element).
#include <cuda_runtime.h>

#include <cstdint>
#include <algorithm>
#include <cstdlib>
#include <utility>

#include "kernels.h"
#include "rf_terms.cuh"

#ifndef BCG_RF_PART
#error "recursion_fact.cu is compiled once per BCG_RF_PART (0..6), see _build.py"
#endif

namespace bcg {

// rf:: term tables: rf_terms.cuh

// cp.async (LDGSTS) helpers
__device__ __forceinline__ void cp_async8(void *dst, const void *src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void *dst, const void *src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// acc[row] -= f1[row offset in S] * f2[row offset in REST] for every register row
template <bool LDG>
__device__ __forceinline__ double ld_factor(const double *p) {
  if constexpr (LDG) {
    return __ldg(p);
  } else {
    return *p;
  }
}
// LDG1 / LDG2: factor read through the read-only global path (else: a plain
// load, shared memory where the factor tensor is resident there)
template <int M, int B, int CT, int S, bool LDG1, bool LDG2, int... Rs>
__device__ __forceinline__ void rows_fma(double *acc, const double *f1, const double *f2,
                                         std::integer_sequence<int, Rs...>) {
  constexpr int REST = ((1 << M) - 1) & ~S;
  ((acc[Rs] = fma(-ld_factor<LDG1>(f1 + rf::HeadOff<S, M, CT, B, Rs>::value),
                  ld_factor<LDG2>(f2 + rf::HeadOff<REST, M, CT, B, Rs>::value), acc[Rs])),
   ...);
}

// Thread <-> (output block, trailing index c): the block is viewed as ROWS x W
// with the leading M-CT modes as rows and the trailing CT modes as columns.
// Lanes take consecutive columns (coalesced M_m / C_m traffic; factor loads are
// broadcast or contiguous across the warp), each thread keeps its ROWS
// elements in registers, and the row offsets into every factor are
// compile-time immediates.
template <int M, int B, int CT, int T>
__device__ __forceinline__ void apply_term(double (&acc)[rf::ipow(B, M - CT)], const int (&dig)[M],
                                           const RecFactArgs &a, const int32_t *toff) {
  constexpr int S = rf::term_mask(M, T);
  constexpr int FULL = (1 << M) - 1;
  constexpr int REST = FULL & ~S;
  constexpr int s = rf::popc(S), r = M - s;
  constexpr int ROWS = rf::ipow(B, M - CT);
  // runtime part: the thread's trailing digits
  int o1 = 0, o2 = 0;
#pragma unroll
  for (int q = M - CT; q < M; ++q) {
    if (S & (1 << q)) o1 += dig[q] * rf::stride_in(S, q, B);
    if (REST & (1 << q)) o2 += dig[q] * rf::stride_in(REST, q, B);
  }
  const double *f1 = a.cum[s] + toff[2 * T] + o1;
  const double *f2 = (r <= 3 ? a.cum[r] : a.cmom[r]) + toff[2 * T + 1] + o2;
  rows_fma<M, B, CT, S, true, true>(acc, f1, f2, std::make_integer_sequence<int, ROWS>{});
}

template <int M, int B, int CT, int... Ts>
__device__ __forceinline__ void apply_terms(double (&acc)[rf::ipow(B, M - CT)], const int (&dig)[M],
                                            const RecFactArgs &a, const int32_t *toff,
                                            std::integer_sequence<int, Ts...>) {
  (apply_term<M, B, CT, Ts>(acc, dig, a, toff), ...);
}

constexpr int kRfThreads = 128;

#ifndef BCG_RF_STREAM
#define BCG_RF_STREAM 1  // cfg5 14.0 -> 13.5 ms (profiles/r01_recursion_res.log)
#endif
template <int M, int B, int CT>
__global__ void __launch_bounds__(kRfThreads, (rf::ipow(B, M - CT) > 32 ? 3 : 4)) k_recursion_fact(RecFactArgs a) {
  constexpr int NT = rf::term_count(M);
  constexpr int ROWS = rf::ipow(B, M - CT);  // elements per thread (registers)
  constexpr int W = rf::ipow(B, CT);         // threads per block
  constexpr int KPC = (kRfThreads + W - 1) / W + 1;  // max output blocks per step
  __shared__ int32_t s_toff[KPC * 2 * NT];
  // each CTA walks a contiguous run of steps (128 items each): consecutive
  // output blocks share most factor blocks, which then stay in this SM's L1.
  // 32-bit item space: the host launches at most 2^31 items at a time.
  const uint32_t nsteps = (uint32_t)((a.nkeys * W + kRfThreads - 1) / kRfThreads);
  const uint32_t s_begin = (uint32_t)((uint64_t)nsteps * blockIdx.x / gridDim.x);
  const uint32_t s_end = (uint32_t)((uint64_t)nsteps * (blockIdx.x + 1) / gridDim.x);
  for (uint32_t step = s_begin; step < s_end; ++step) {
    const uint32_t item0 = step * kRfThreads;
    const uint32_t kb0 = item0 / W;
    __syncthreads();  // previous step done with s_toff
    // stage the term-offset rows of this step's output blocks: one contiguous
    // run of the work-list-ordered table (coalesced, no key indirection), so
    // every factor address below is a shared-memory read away
    {
      const int32_t *src = a.term_off + (int64_t)kb0 * 2 * NT;
      const int64_t left = (a.nkeys - (int64_t)kb0) * 2 * NT;
      const int lim = left < KPC * 2 * NT ? (int)left : KPC * 2 * NT;
      for (int i = threadIdx.x; i < lim; i += kRfThreads) s_toff[i] = __ldg(src + i);
    }
    __syncthreads();
    const int rel = (int)(item0 - kb0 * W) + threadIdx.x;  // item offset from block kb0's first item
    const int kbr = rel / W;                                  // W is a compile-time constant
    const int64_t kb = (int64_t)kb0 + kbr;
    if (kb >= a.nkeys) continue;
    const int c = rel - kbr * W;
    const int32_t *toff = s_toff + kbr * 2 * NT;
    int dig[M];
#pragma unroll
    for (int q = 0; q < M; ++q) dig[q] = 0;
    {
      int rem = c;
#pragma unroll
      for (int q = M - 1; q >= M - CT; --q) {
        dig[q] = rem % B;
        rem /= B;
      }
    }
    double *blk = a.mk + __ldg(a.blk_off + kb) + c;
    double acc[ROWS];
#pragma unroll
#if BCG_RF_STREAM
    // M_m is read once and C_m written once: streaming (evict-first) accesses
    // keep them from displacing the factor blocks the neighbouring outputs
    // re-read from L1
    for (int row = 0; row < ROWS; ++row) acc[row] = __ldcs(blk + (int64_t)row * W);
#else
    for (int row = 0; row < ROWS; ++row) acc[row] = blk[(int64_t)row * W];
#endif
    apply_terms<M, B, CT>(acc, dig, a, toff, std::make_integer_sequence<int, NT>{});
#pragma unroll
#if BCG_RF_STREAM
    for (int row = 0; row < ROWS; ++row) __stcs(blk + (int64_t)row * W, acc[row]);
#else
    for (int row = 0; row < ROWS; ++row) blk[(int64_t)row * W] = acc[row];
#endif
  }
}

// v6 (m = 6, 3 <= b <= 7): one CTA per output block, walked in B slabs of
// fixed mode-1 index i0.  Every term's second factor (the modes NOT holding
// mode 1: central moment / cumulant of the complement) is the same for all
// slabs, so it is staged in shared memory ONCE per block; the first factor's
// slice at i0 (a contiguous run: mode 1 is its leading mode) is staged per
// slab, double-buffered by cp.async while the previous slab is evaluated.  All
// factor reads are then LDS (v2 reads them through L1 at ~3 wavefronts per
// request and re-fetches them from L2: 50 GB of L2->L1 traffic per 20 GB of
// M_6 at cfg5).  Within a slab (modes 2..6): modes 2, 3 in registers (B^2
// rows), modes 4..6 across threads (B^3, coalesced M_m / C_m rows).
template <int B>
struct Slab6 {
  static constexpr int M = 6;
  static constexpr int NT = rf::term_count(M);
  static constexpr int CT = 3;                    // thread modes of the 5-mode slab
  static constexpr int ROWS = B * B;
  static constexpr int W = B * B * B;
  static constexpr int NTH = (W + 31) / 32 * 32;
  static constexpr int SLAB = B * B * B * B * B;  // elements per slab
  // second factors (no mode 1), all terms: offset of term T
  __host__ __device__ static constexpr int ov(int T) {
    int o = 0;
    for (int t = 0; t < T; ++t) o += rf::ipow(B, M - rf::popc(rf::term_mask(M, t)));
    return o;
  }
  // first-factor slices (mode 1 fixed): offset of term T
  __host__ __device__ static constexpr int ou(int T) {
    int o = 0;
    for (int t = 0; t < T; ++t) o += rf::ipow(B, rf::popc(rf::term_mask(M, t)) - 1);
    return o;
  }
  static constexpr int SEGV = ov(NT), SEGU = (ou(NT) + 1) / 2 * 2;
  // slabs evaluated concurrently (thread groups): two where the CTA stays <= 1024
  // threads and the stages fit
  static constexpr int G = (2 * NTH <= 1024 && (SEGV + 4 * SEGU) * 8 <= 200 * 1024) ? 2 : 1;
  static constexpr size_t SMEM = (size_t)(SEGV + 2 * G * SEGU) * 8;
  static constexpr bool ok = B >= 3 && B <= 7 && SMEM <= 200 * 1024;
};

template <int B, int T>
__device__ __forceinline__ void slab6_stage_v(double *sv, const RecFactArgs &a, const int32_t *toff, int tid) {
  using SL = Slab6<B>;
  constexpr int S = rf::term_mask(6, T);
  constexpr int r = 6 - rf::popc(S);
  constexpr int L = rf::ipow(B, r);
  const double *src = (r <= 3 ? a.cum[r] : a.cmom[r]) + __ldg(toff + 2 * T + 1);
  for (int i = tid; i < L; i += SL::NTH) cp_async8(sv + std::integral_constant<int, SL::ov(T)>::value + i, src + i);
}
template <int B, int T>
__device__ __forceinline__ void slab6_stage_u(double *su, const RecFactArgs &a, const int32_t *toff, int i0, int tid) {
  using SL = Slab6<B>;
  constexpr int S = rf::term_mask(6, T);
  constexpr int s = rf::popc(S);
  constexpr int L = rf::ipow(B, s - 1);  // the slice of the C_s block at mode-1 index i0
  const double *src = a.cum[s] + __ldg(toff + 2 * T) + i0 * L;
  for (int i = tid; i < L; i += SL::NTH) cp_async8(su + std::integral_constant<int, SL::ou(T)>::value + i, src + i);
}
template <int B, int... Ts>
__device__ __forceinline__ void slab6_stage_v_all(double *sv, const RecFactArgs &a, const int32_t *toff, int tid,
                                                  std::integer_sequence<int, Ts...>) {
  (slab6_stage_v<B, Ts>(sv, a, toff, tid), ...);
}
template <int B, int... Ts>
__device__ __forceinline__ void slab6_stage_u_all(double *su, const RecFactArgs &a, const int32_t *toff, int i0,
                                                  int tid, std::integer_sequence<int, Ts...>) {
  (slab6_stage_u<B, Ts>(su, a, toff, i0, tid), ...);
}

// term T on a slab: the 5-mode problem over original modes 1..5 (bit q of a
// slab mask = original mode q+1), u over A = S \ {0}, v over the rest
template <int B, int T>
__device__ __forceinline__ void slab6_term(double (&acc)[Slab6<B>::ROWS], const int (&dig)[5], const double *su,
                                           const double *sv) {
  using SL = Slab6<B>;
  constexpr int S = rf::term_mask(6, T);
  constexpr int A = S >> 1;                   // slab modes of the first factor
  constexpr int R = (((1 << 6) - 1) & ~S) >> 1;  // slab modes of the second factor
  int o1 = 0, o2 = 0;
#pragma unroll
  for (int q = 5 - SL::CT; q < 5; ++q) {
    if (A & (1 << q)) o1 += dig[q] * rf::stride_in(A, q, B);
    if (R & (1 << q)) o2 += dig[q] * rf::stride_in(R, q, B);
  }
  rows_fma<5, B, SL::CT, A, false, false>(acc, su + std::integral_constant<int, SL::ou(T)>::value + o1,
                                          sv + std::integral_constant<int, SL::ov(T)>::value + o2,
                                          std::make_integer_sequence<int, SL::ROWS>{});
}
template <int B, int... Ts>
__device__ __forceinline__ void slab6_terms(double (&acc)[Slab6<B>::ROWS], const int (&dig)[5], const double *su,
                                            const double *sv, std::integer_sequence<int, Ts...>) {
  (slab6_term<B, Ts>(acc, dig, su, sv), ...);
}

// G slabs are evaluated at once by G thread groups sharing the staged second
// factors (1 CTA/SM: 14 warps at b = 6 instead of 7).
template <int B>
__global__ void __launch_bounds__(Slab6<B>::NTH * Slab6<B>::G) k_recursion_slab6(RecFactArgs a) {
  using SL = Slab6<B>;
  constexpr int G = SL::G;
  extern __shared__ __align__(16) unsigned char rf_smem[];
  double *sv = reinterpret_cast<double *>(rf_smem);
  double *su = sv + SL::SEGV;  // [2 stages][G groups][SEGU]
  const int tid = threadIdx.x % SL::NTH, grp = threadIdx.x / SL::NTH;
  const int64_t kb = blockIdx.x;
  const int32_t *toff = a.term_off + kb * 2 * SL::NT;
  slab6_stage_v_all<B>(sv, a, toff, tid + grp * SL::NTH, std::make_integer_sequence<int, SL::NT>{});
  if (grp < B) slab6_stage_u_all<B>(su + grp * SL::SEGU, a, toff, grp, tid, std::make_integer_sequence<int, SL::NT>{});
  cp_async_commit();
  const bool active = tid < SL::W;
  const int c = active ? tid : 0;
  int dig[5];
  dig[0] = dig[1] = 0;
  dig[2] = c / (B * B);
  dig[3] = (c / B) % B;
  dig[4] = c % B;
  double *blk = a.mk + __ldg(a.blk_off + kb) + c;
  constexpr int ROUNDS = (B + G - 1) / G;
#pragma unroll 1
  for (int rd = 0; rd < ROUNDS; ++rd) {
    const int i0 = rd * G + grp;
    const int nx = i0 + G;  // this group's slab of the next round
    if (nx < B)
      slab6_stage_u_all<B>(su + (((rd + 1) & 1) * G + grp) * SL::SEGU, a, toff, nx, tid,
                           std::make_integer_sequence<int, SL::NT>{});
    cp_async_commit();
    const bool live = active && i0 < B;
    double acc[SL::ROWS];
    double *row = blk + (int64_t)i0 * SL::SLAB;
    if (live) {
#pragma unroll
      for (int r = 0; r < SL::ROWS; ++r) acc[r] = row[r * SL::W];
    }
    cp_async_wait<1>();  // V and this round's U slices have landed (this thread's copies)
    __syncthreads();     // ... everyone's
    if (live) {
      slab6_terms<B>(acc, dig, su + ((rd & 1) * G + grp) * SL::SEGU, sv, std::make_integer_sequence<int, SL::NT>{});
#pragma unroll
      for (int r = 0; r < SL::ROWS; ++r) row[r * SL::W] = acc[r];
    }
    __syncthreads();  // this round's U buffers are restaged two rounds on
  }
}

// trailing (thread) modes: the fewest that leave <= kRfRows register rows
#ifndef BCG_RF_ROWS
#define BCG_RF_ROWS 32
#endif
__host__ __device__ constexpr int ct_for(int M, int B) {
  int c = 0;
  while (c < M && rf::ipow(B, M - c) > BCG_RF_ROWS) ++c;
  return c;
}

// ---------------------------------------------------------------------------
// v3: one CTA per output block, every factor sub-block of the block staged in
// shared memory first (sizes and offsets compile-time), then the same
// register-blocked evaluation reading shared memory only.  Used when the
// staged factors fit in 48 KB; otherwise v2 above (factors through L1).
namespace rf {
// doubles of factor storage for terms < T (both factors of each term)
__host__ __device__ constexpr int seg_before(int M, int B, int T) {
  int off = 0;
  for (int t = 0; t < T; ++t) {
    const int sz = popc(term_mask(M, t));
    off += ipow(B, sz) + ipow(B, M - sz);
  }
  return off;
}
// staged thread modes: at least 64 threads, at most 32 register rows
__host__ __device__ constexpr int ct_staged(int M, int B) {
  int c1 = 0;
  while (c1 < M - 1 && ipow(B, c1) < 64) ++c1;
  int c2 = 0;
  while (c2 < M && ipow(B, M - c2) > 32) ++c2;
  return c1 > c2 ? c1 : c2;
}
}  // namespace rf

template <int M, int B>
struct Staged {
  static constexpr int NT = rf::term_count(M);
  static constexpr int CT = rf::ct_staged(M, B);
  static constexpr int W = rf::ipow(B, CT);
  static constexpr int ROWS = rf::ipow(B, M - CT);
  static constexpr int NTH = (W + 31) / 32 * 32;
  static constexpr int SEG = rf::seg_before(M, B, NT);
  // staging pays off when the factor sub-blocks are no larger than the
  // output block itself (cfg2, cfg3; cfg4's 25 terms stage 2.6x the block)
  static constexpr bool fits = SEG * 8 <= 48 * 1024 && NTH <= 1024 && ROWS <= 32;
  static constexpr bool ok = fits && SEG <= rf::ipow(B, M);
};

template <int M, int B, int T>
__device__ __forceinline__ void stage_term(double *sm, const RecFactArgs &a, const int32_t *toff, int tid) {
  constexpr int S = rf::term_mask(M, T);
  constexpr int s = rf::popc(S), r = M - s;
  constexpr int L1 = rf::ipow(B, s), L2 = rf::ipow(B, r);
  constexpr int O1 = rf::seg_before(M, B, T), O2 = O1 + L1;
  constexpr int NTH = Staged<M, B>::NTH;
  const double *src1 = a.cum[s] + toff[2 * T];
  const double *src2 = (r <= 3 ? a.cum[r] : a.cmom[r]) + toff[2 * T + 1];
  for (int i = tid; i < L1; i += NTH) sm[O1 + i] = __ldg(src1 + i);
  for (int i = tid; i < L2; i += NTH) sm[O2 + i] = __ldg(src2 + i);
}

template <int M, int B, int T>
__device__ __forceinline__ void apply_term_staged(double (&acc)[Staged<M, B>::ROWS], const int (&dig)[M],
                                                  const double *sm) {
  constexpr int CT = Staged<M, B>::CT, ROWS = Staged<M, B>::ROWS;
  constexpr int S = rf::term_mask(M, T);
  constexpr int REST = ((1 << M) - 1) & ~S;
  constexpr int s = rf::popc(S);
  constexpr int O1 = rf::seg_before(M, B, T), O2 = O1 + rf::ipow(B, s);
  int o1 = 0, o2 = 0;
#pragma unroll
  for (int q = M - CT; q < M; ++q) {
    if (S & (1 << q)) o1 += dig[q] * rf::stride_in(S, q, B);
    if (REST & (1 << q)) o2 += dig[q] * rf::stride_in(REST, q, B);
  }
  const double *f1 = sm + O1 + o1;
  const double *f2 = sm + O2 + o2;
  rows_fma<M, B, CT, S, false, false>(acc, f1, f2, std::make_integer_sequence<int, ROWS>{});
}

template <int M, int B, int... Ts>
__device__ __forceinline__ void staged_all(double *sm, double (&acc)[Staged<M, B>::ROWS], const int (&dig)[M],
                                           const RecFactArgs &a, const int32_t *toff, int tid, bool active,
                                           std::integer_sequence<int, Ts...>) {
  (stage_term<M, B, Ts>(sm, a, toff, tid), ...);
  __syncthreads();
  if (active) (apply_term_staged<M, B, Ts>(acc, dig, sm), ...);
}

template <int M, int B>
__global__ void __launch_bounds__(Staged<M, B>::NTH) k_recursion_staged(RecFactArgs a) {
  using ST = Staged<M, B>;
  __shared__ double sm[ST::SEG];
  const int tid = threadIdx.x;
  const int32_t *toff = a.term_off + (int64_t)blockIdx.x * 2 * ST::NT;
  const bool active = tid < ST::W;
  const int c = active ? tid : 0;
  int dig[M];
#pragma unroll
  for (int q = 0; q < M; ++q) dig[q] = 0;
  {
    int rem = c;
#pragma unroll
    for (int q = M - 1; q >= M - ST::CT; --q) {
      dig[q] = rem % B;
      rem /= B;
    }
  }
  double *blk = a.mk + a.blk_off[blockIdx.x] + c;
  double acc[ST::ROWS];
  // M_m first: its HBM latency overlaps the factor staging
#pragma unroll
  for (int row = 0; row < ST::ROWS; ++row) acc[row] = active ? blk[(int64_t)row * ST::W] : 0.0;
  staged_all<M, B>(sm, acc, dig, a, toff, tid, active, std::make_integer_sequence<int, ST::NT>{});
  if (active) {
#pragma unroll
    for (int row = 0; row < ST::ROWS; ++row) blk[(int64_t)row * ST::W] = acc[row];
  }
}

#if BCG_RF_PART == 0
// ---- part 0: dispatch (the (m, b) instantiations live in parts 1..6,
// separate translation units so nvcc compiles them in parallel) ----
template <int M, int B>
cudaError_t go_fact(const RecFactArgs &a, cudaStream_t stream);

int recursion_fact_terms(int m) { return rf::term_count(m); }

bool recursion_fact_supported(int m, int b) { return m >= 4 && m <= 6 && b >= 1 && b <= 8; }

cudaError_t launch_recursion_fact(const RecFactArgs &a, int m, int b, cudaStream_t stream) {
#define RF_B(M)                                    \
  switch (b) {                                     \
    case 1: return go_fact<M, 1>(a, stream);       \
    case 2: return go_fact<M, 2>(a, stream);       \
    case 3: return go_fact<M, 3>(a, stream);       \
    case 4: return go_fact<M, 4>(a, stream);       \
    case 5: return go_fact<M, 5>(a, stream);       \
    case 6: return go_fact<M, 6>(a, stream);       \
    case 7: return go_fact<M, 7>(a, stream);       \
    case 8: return go_fact<M, 8>(a, stream);       \
    default: return cudaErrorInvalidValue;         \
  }
  switch (m) {
    case 4: RF_B(4)
    case 5: RF_B(5)
    case 6: RF_B(6)
    default: return cudaErrorInvalidValue;
  }
#undef RF_B
}
#else
template <int M, int B, int CT>
static cudaError_t go_fact_v2(const RecFactArgs &a_in, cudaStream_t stream) {
  constexpr int W = rf::ipow(B, CT);
  // the kernel's item arithmetic is 32-bit: launch key chunks of < 2^31 items
  constexpr int64_t kMaxKeys = ((int64_t)1 << 31) / W - 1;
  RecFactArgs a = a_in;
  while (a.nkeys > kMaxKeys) {
    RecFactArgs part = a;
    part.nkeys = kMaxKeys;
    cudaError_t e = go_fact_v2<M, B, CT>(part, stream);
    if (e != cudaSuccess) return e;
    a.blk_off += kMaxKeys;
    a.term_off += kMaxKeys * 2 * rf::term_count(M);
    a.nkeys -= kMaxKeys;
  }
  const int64_t steps = (a.nkeys * W + kRfThreads - 1) / kRfThreads;
  if (steps <= 0) return cudaSuccess;
  static const int per_cta = getenv("BCG_RF_STEPS") ? atoi(getenv("BCG_RF_STEPS")) : 1;  // tuning knob
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(steps, (steps + per_cta - 1) / per_cta));
  k_recursion_fact<M, B, CT><<<(unsigned)blocks, kRfThreads, 0, stream>>>(a);
  g_launches++;
  return cudaGetLastError();
}

template <int M, int B>
cudaError_t go_fact(const RecFactArgs &a, cudaStream_t stream) {
  // A/B knob: BCG_RF_VARIANT=2 (v2), 3 (v3 staged), 6 (v6 slab-staged, m = 6), 7 (v7 streamed, m = b = 6)
  static const int variant = getenv("BCG_RF_VARIANT") ? atoi(getenv("BCG_RF_VARIANT")) : 0;
  static const bool no_staged = getenv("BCG_RF_NO_STAGED") != nullptr || variant == 2 || variant == 6;
  if constexpr (M == 6 && B == 6) {
    // v7 (recursion_stream.cu): bulk-copy streamed, default where every
    // factor / block pointer is 16-byte aligned
    if (variant == 0 || variant == 7) {
      bool aligned = ((uintptr_t)a.mk & 15) == 0;
      for (int k = 2; k <= 4; ++k) aligned = aligned && ((uintptr_t)a.cum[k] & 15) == 0;
      aligned = aligned && ((uintptr_t)a.cmom[4] & 15) == 0;
      if (aligned) return launch_recursion_stream6(a, B, stream);
    }
  }
  if constexpr (M == 6 && Slab6<B>::ok) {
    if (variant == 6) {  // measured equal to v2 at cfg5, slower at cfg4 (profiles/r01_recursion_ncu.txt)
      if (a.nkeys <= 0) return cudaSuccess;
      using SL = Slab6<B>;
      // per launch: the attribute is per device
      cudaError_t e = cudaFuncSetAttribute(k_recursion_slab6<B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)SL::SMEM);
      if (e != cudaSuccess) return e;
      k_recursion_slab6<B><<<(unsigned)a.nkeys, SL::NTH * SL::G, SL::SMEM, stream>>>(a);
      g_launches++;
      return cudaGetLastError();
    }
  }
  if constexpr (Staged<M, B>::fits) {
    if (Staged<M, B>::ok ? !no_staged : variant == 3) {
      if (a.nkeys <= 0) return cudaSuccess;
      k_recursion_staged<M, B><<<(unsigned)a.nkeys, Staged<M, B>::NTH, 0, stream>>>(a);
      g_launches++;
      return cudaGetLastError();
    }
  }
  constexpr int CT = ct_for(M, B);
  // A/B knob BCG_RF_TILE=+1: one more leading mode in registers (where it stays
  // <= 64 rows), -1: one fewer
  constexpr int CTW = (CT > 1 && rf::ipow(B, M - CT + 1) <= 64) ? CT - 1 : CT;
  constexpr int CTN = CT < M - 1 ? CT + 1 : CT;
  // default: the wider tile when the narrow one keeps fewer than 16 rows
  // (b = 6, m = 6: 6 -> 36 rows, 1.9x faster at the cfg5 layout)
  static const int tile = getenv("BCG_RF_TILE") ? atoi(getenv("BCG_RF_TILE")) : (rf::ipow(B, M - CT) < 16 ? 1 : 0);
  if (tile > 0 && CTW != CT) return go_fact_v2<M, B, CTW>(a, stream);
  if (tile < 0 && CTN != CT) return go_fact_v2<M, B, CTN>(a, stream);
  return go_fact_v2<M, B, CT>(a, stream);
}

#define RF_INST(M, B) template cudaError_t go_fact<M, B>(const RecFactArgs &, cudaStream_t);
#if BCG_RF_PART == 1
RF_INST(4, 1) RF_INST(4, 2) RF_INST(4, 3) RF_INST(4, 4) RF_INST(4, 5) RF_INST(4, 6) RF_INST(4, 7) RF_INST(4, 8)
#elif BCG_RF_PART == 2
RF_INST(5, 1) RF_INST(5, 2) RF_INST(5, 3) RF_INST(5, 4)
#elif BCG_RF_PART == 3
RF_INST(5, 5) RF_INST(5, 6) RF_INST(5, 7) RF_INST(5, 8)
#elif BCG_RF_PART == 4
RF_INST(6, 1) RF_INST(6, 2) RF_INST(6, 3)
#elif BCG_RF_PART == 5
RF_INST(6, 4) RF_INST(6, 5) RF_INST(6, 6)
#elif BCG_RF_PART == 6
RF_INST(6, 7) RF_INST(6, 8)
#endif
#undef RF_INST
#endif  // BCG_RF_PART

}  // namespace bcg
