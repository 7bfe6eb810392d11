// K3 (v7 .. v9): order-6 cumulant recursion streamed by the bulk-copy engine,
// for full blocks of edge b = 6 (the cfg5 layout).
//
// Same arithmetic as v2 (recursion_fact.cu, the factored form of the
// reference's partition sum bc/cumulants.py:53-136):
//
//   C_6 = M_6 - sum_{S containing mode 0, 2 <= |S| <= 4} C_|S|[key|S] * M_{6-|S|}[key|rest]
//
// 25 terms, applied per element in the same order with the same fma(-f1, f2, acc)
// as v2, so both kernels produce bitwise-identical C_6.
//
// Why: v2 reads its factors through L1 (50 GB of L2->L1 traffic per 20 GB of
// M_6 at cfg5, 53% L1 hit, long-scoreboard stalls).  Here:
//
//   * persistent CTAs, one per SM, each over a contiguous run of the work
//     list; the host orders the list by the key's modes 1..5 ("tail"), and
//     blocks with equal tails share all 25 second factors;
//   * a block is b slabs (mode-0 index i0), a slab b sub-slabs (mode-1 index
//     i1) of b^4 elements; a "unit" is 2 sub-slabs (20.7 KB at b = 6), one
//     contiguous run of M_6;
//   * warp 0 streams units into an NS-stage shared-memory ring
//     (cp.async.bulk, mbarrier complete_tx) and prefetches ahead into L2;
//   * warp 1 streams the factors, one lane per term (a V or U load is ONE
//     warp-wide bulk-copy instruction): per tail the 25 second factors (V: the
//     sub-blocks not holding mode 0, 72 KB at b = 6), per slab the 25
//     first-factor slices at i0 (U: 20 KB, NU buffers); M_6 copies carry an
//     L2 evict-first policy, factor copies evict-last;
//   * NGRP (4) consumer groups of 3 warps: a group loads a unit's elements from its ring
//     stage into registers and releases the stage at once, applies the 25
//     terms reading the factors from shared memory (v9: 81 of a thread's 364
//     factor values per unit from its tensor-memory lane instead, see "tensor
//     memory" below), and stores C_6 straight from registers to HBM
//     (streaming stores, in place over M_6).
//
// Register tile: a thread owns (b/2)^NRM elements: b/2 digits of each of
// the NRM trailing modes, interleaved with 2 thread groups per mode
// (index = 2 d + g), the other modes 2.. at thread level.  Splitting every
// mode's range between registers and threads makes each term's two factors
// split the tile (loads per term = 3^|S & tile| + 3^|rest & tile|): 0.33
// (NRM = 4, 81 elements) / 0.54 (NRM = 3, 27 elements) shared-memory loads per
// FMA, against v2's 0.64.  Interleaving keeps g5 lanes on adjacent doubles, so
// a warp's store touches 16-byte runs, and the 16 lanes of a sub-slab hit
// distinct double-banks on the ring loads.
//
// Lane order (v8).  ncu's per-instruction wavefront counts of v7d fit one rule
// exactly (tools/rs_wavefront_model.py, profiles/r02_rs_wavefront_rule.txt):
// an LDS.64 whose lane quads each read <= 2 distinct addresses takes the bank
// rule over the warp, any other the sum of its two half-warps' bank rules -- a
// factor indexed by BOTH lane bits 0 and 1 costs two wavefronts even when the
// warp reads 4 distinct doubles.  v8 puts the low bit of the mode-2 digit and
// the sub-slab in lane bits 0, 1 (0.476 factor wavefronts per element instead
// of 0.633, as ncu then measured; tools/lds_rate.cu confirms on the hardware
// that an LDS.64 costs its wavefronts, 1 cycle per SM each).  That changed the
// time by 0.3%: shared-memory bandwidth is not what bounds the consumers (L1
// data pipe 65% busy, FP64 pipe 37%, issue slots 40% in ncu) -- they run
// dependent LDS -> DFMA chains at 3 warps per scheduler and 128 registers.
// A larger register tile (fewer loads per FMA) does not fit: at b = 6 = 2 x 3
// the 27-element tile is the only one whose thread count per unit is a
// multiple of 32 short of 81 elements (254 registers, measured slower); a
// fifth consumer group (15 warps) measured no faster.
//
// mbarrier phases: consumers release ring stages early and run ahead of each
// other, so a "full" barrier is indexed such that its previous phase belongs
// to the same consumer group (which has observed it complete): unit u ->
// stage u % NS, full barrier u % lcm(NS, NGRP); slab s -> U buffer s % NU,
// full barrier s % lcm(NU, slab period).  Otherwise a parity wait could pass
// on a phase two behind.
//
// Roofline: HBM, 16 B per element (M_6 in, C_6 out) + every factor value once
// per tail / slab (from L2).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <utility>

#include "kernels.h"
#include "kr.cuh"  // BCG_CHECK
#include "rf_terms.cuh"

namespace bcg {

namespace rs {

using rf::ipow;
using rf::popc;
using rf::stride_in;
using rf::term_count;
using rf::term_mask;

constexpr int gcd(int x, int y) { return y == 0 ? x : gcd(y, x % y); }
constexpr int lcm(int x, int y) { return x / gcd(x, y) * y; }

// geometry for order 6, edge B, NRM register modes (the trailing ones),
// NGRP consumer groups
template <int B, int RM, int NGRP, int NU_ = 3, int XB = 1, int LO_ = 0, int HINT_ = 0, int PP_ = 0, int TM_ = 0>
struct Geo {
  static constexpr int TM = TM_;      // 1: tail-constant second factors cached per lane in tensor memory
  static constexpr int PP = PP_;      // factor producer: 0 = one lane issues all copies, 1 = one lane per term
  static constexpr int LO = LO_;      // consumer lane order (see the kernel)
  static constexpr int HINT = HINT_;  // L2 eviction hints on the bulk copies
  static constexpr int M = 6;
  static constexpr int NT = term_count(M);  // 25
  static constexpr int RG = B / 2;          // register digits per register mode
  static constexpr int NRM = popc(RM);      // register modes (a subset of 2..5)
  static constexpr int TPS = ipow(B, 4 - NRM) * ipow(2, NRM);  // threads per sub-slab
  static constexpr int U1 = 2;                                 // sub-slabs per unit
  static constexpr int GT = U1 * TPS;                          // threads per group
  static constexpr int GW = GT / 32;                           // warps per group
  static constexpr int ROWS = ipow(RG, NRM);                   // elements per thread
  static constexpr int SUB = ipow(B, 4);                       // elements per sub-slab
  static constexpr int UNIT = U1 * SUB;                        // elements per unit
  static constexpr int UPS = B / U1;                           // units per slab
  static constexpr int UPB = B * UPS;                          // units per block
  static constexpr int NU = NU_;                               // U buffers
  // PP = 2: ONE producer warp (lane 31 streams M_6, lanes 0..24 the factors),
  // so 5 consumer groups fit 512 threads at 128 registers
  static constexpr int PW = PP_ == 2 ? 1 : 2;  // producer warps
  static constexpr int NTHREADS = 32 * PW + NGRP * GT;
  // second factor of term T (modes not holding 0): b^|rest| doubles at ov(T)
  __host__ __device__ static constexpr int ov(int T) {
    int o = 0;
    for (int t = 0; t < T; ++t) o += ipow(B, M - popc(term_mask(M, t)));
    return o;
  }
  // first factor of term T sliced at i0: b^(|S|-1) doubles at ou(T)
  __host__ __device__ static constexpr int ou(int T) {
    int o = 0;
    for (int t = 0; t < T; ++t) o += ipow(B, popc(term_mask(M, t)) - 1);
    return o;
  }
  static constexpr int SEGV = ov(NT), SEGU = ou(NT);
  // units go round-robin to the groups, so the pattern of slabs a group
  // visits repeats every NGRP / gcd(NGRP, UPS) slabs; a U full barrier period
  // that is a multiple of it means a group waiting on slab s has also waited
  // on slab s - UF, the barrier's previous phase
  static constexpr int SLAB_PERIOD = NGRP / gcd(NGRP, UPS);
  static constexpr int NS = (227 * 1024 - 8 * (SEGV + NU * SEGU) - 512) / (8 * UNIT);  // ring stages
  static constexpr int MF = lcm(NS, NGRP) * XB;
  static constexpr int UF = lcm(NU, SLAB_PERIOD) * XB;
  static constexpr int NBAR = MF + NS + UF + NU + 2 + 2;  // + done barrier, TMEM base slot
  static constexpr size_t SMEM = 8 * (size_t)(SEGV + NU * SEGU + NS * UNIT) + 8 * NBAR;
  // every bulk copy is a multiple of 16 bytes at a 16-byte aligned offset
  static constexpr bool ok = B % 2 == 0 && B >= 4 && GT % 32 == 0 && NS >= 2 && SEGU % 2 == 0 &&
                             UNIT % 2 == 0 && SMEM <= 227 * 1024;
};

// element offset, inside the factor over the modes of MASK (row-major), of
// the register digits of tile row ROW (digits of the modes in RM, the last
// fastest; index = 2 d + g)
template <int MASK, int B, int RM, int ROW>
struct RowOff {
  static constexpr int calc() {
    int off = 0, r = ROW;
    for (int q = 5; q >= 2; --q) {
      if (!(RM & (1 << q))) continue;
      const int d = r % (B / 2);
      r /= B / 2;
      if (MASK & (1 << q)) off += 2 * d * stride_in(MASK, q, B);
    }
    return off;
  }
  static constexpr int value = calc();
};

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void bar_init(uint64_t *b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void bar_wait(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "RS_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra.uni RS_DONE;\n"
      "bra.uni RS_WAIT;\n"
      "RS_DONE:\n"
      "}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
// the same for a warp whose lanes wait on different barriers (PP = 2: the
// M_6 lane and the factor lanes share a warp): no uniform branches, and
// test_wait, not try_wait -- a try_wait suspends the whole warp, the other
// lanes' path with it, until its time limit
__device__ __forceinline__ void bar_wait_div(uint64_t *b, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(ok)
        : "r"(su32(b)), "r"(parity)
        : "memory");
    if (!ok) __nanosleep(32);  // let the warp's other path run
  } while (!ok);
}
__device__ __forceinline__ void bar_expect(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
// global -> shared bulk copy completing on an mbarrier
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(b))
      : "memory");
}
// the same with an L2 eviction-priority policy (createpolicy)
__device__ __forceinline__ void bulk_g2s_hint(void *dst, const void *src, uint32_t bytes, uint64_t *b, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(b)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
// bulk prefetch into L2 (no shared memory)
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}

// ---- factor producer ----
template <class G, int T>
__device__ __forceinline__ void load_v(double *sv, const RecFactArgs &a, const int32_t *toff, uint64_t *bar,
                                       uint64_t pol) {
  constexpr int r = 6 - popc(term_mask(6, T));
  constexpr int B = 2 * G::RG;
  const double *src = (r <= 3 ? a.cum[r] : a.cmom[r]) + __ldg(toff + 2 * T + 1);
  if constexpr (G::HINT) bulk_g2s_hint(sv + G::ov(T), src, 8u * ipow(B, r), bar, pol);
  else bulk_g2s(sv + G::ov(T), src, 8u * ipow(B, r), bar);
}
template <class G, int T>
__device__ __forceinline__ void load_u(double *su, const RecFactArgs &a, const int32_t *toff, int i0, uint64_t *bar,
                                       uint64_t pol) {
  constexpr int s = popc(term_mask(6, T));
  constexpr int L = ipow(2 * G::RG, s - 1);
  const double *src = a.cum[s] + __ldg(toff + 2 * T) + (int64_t)i0 * L;
  if constexpr (G::HINT) bulk_g2s_hint(su + G::ou(T), src, 8u * L, bar, pol);
  else bulk_g2s(su + G::ou(T), src, 8u * L, bar);
}
template <class G, int... Ts>
__device__ __forceinline__ void load_v_all(double *sv, const RecFactArgs &a, const int32_t *toff, uint64_t *bar,
                                           uint64_t pol, std::integer_sequence<int, Ts...>) {
  (load_v<G, Ts>(sv, a, toff, bar, pol), ...);
}
template <class G, int... Ts>
__device__ __forceinline__ void load_u_all(double *su, const RecFactArgs &a, const int32_t *toff, int i0,
                                           uint64_t *bar, uint64_t pol, std::integer_sequence<int, Ts...>) {
  (load_u<G, Ts>(su, a, toff, i0, bar, pol), ...);
}

// ---- tensor memory as a per-lane operand cache (TM = 1) ----
// Five terms' second factors hold no mode 1, so a thread reads the same 81
// doubles of V in every unit of a tail: they are copied once per tail into
// the warp's tensor-memory lanes (tcgen05.st, 162 columns of a lane per warp;
// 3 consumer warps share a 32-lane quadrant, 486 of 512 columns) and read back
// with 18 tcgen05.ld per unit instead of 81 of the unit's 391 LDS.64 (fewer
// instructions through the LSU queue the consumers stall on; measured -1.5 to
// -4.8%).
__host__ __device__ constexpr bool tm_term(int T) { return T == 0 || T == 2 || T == 4 || T == 6 || T == 8; }
template <int RM>
__host__ __device__ constexpr int tm_vcount(int T) {
  return ipow(3, popc((63 & ~term_mask(6, T)) & RM));
}
template <int RM>
__host__ __device__ constexpr int tm_col(int T) {  // first column (32-bit) of term T's values
  int c = 0;
  for (int t = 0; t < T; ++t)
    if (tm_term(t)) c += 2 * tm_vcount<RM>(t);
  return c;
}
template <int RM>
__host__ __device__ constexpr int tm_cols() { return tm_col<RM>(25); }
// factor offset of the J-th distinct register-digit combination of the modes
// in R (mode 5 fastest), and the combination a tile row uses
template <int R, int B, int RM, int J>
struct VOffJ {
  static constexpr int calc() {
    int off = 0, j = J;
    for (int q = 5; q >= 2; --q) {
      if (!(RM & (1 << q)) || !(R & (1 << q))) continue;
      const int d = j % (B / 2);
      j /= B / 2;
      off += 2 * d * stride_in(R, q, B);
    }
    return off;
  }
  static constexpr int value = calc();
};
template <int R, int B, int RM, int ROW>
struct VJ {
  static constexpr int calc() {
    int j = 0, mul = 1, r = ROW;
    for (int q = 5; q >= 2; --q) {
      if (!(RM & (1 << q))) continue;
      const int d = r % (B / 2);
      r /= B / 2;
      if (R & (1 << q)) {
        j += d * mul;
        mul *= B / 2;
      }
    }
    return j;
  }
  static constexpr int value = calc();
};
__device__ __forceinline__ void tm_st1(uint32_t taddr, double v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};\n" ::"r"(taddr), "r"(__double2loint(v)),
               "r"(__double2hiint(v))
               : "memory");
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
// 9 doubles (18 columns) of the lane; the wait is part of the statement so no
// use of the registers can be scheduled before it
__device__ __forceinline__ void tm_ld9(uint32_t taddr, double (&v)[9]) {
  uint32_t r[18];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%18];\n"
      "tcgen05.ld.sync.aligned.32x32b.x2.b32 {%16, %17}, [%19];\n"
      "tcgen05.wait::ld.sync.aligned;\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17])
      : "r"(taddr), "r"(taddr + 16)
      : "memory");
#pragma unroll
  for (int i = 0; i < 9; ++i) v[i] = __hiloint2double((int)r[2 * i + 1], (int)r[2 * i]);
}
// copy term T's values of this thread (o2 = its offset in the factor) into its lane
template <class G, int B, int RM, int T, int... Js>
__device__ __forceinline__ void tm_fill_term(uint32_t tbase, const double *sv, const int (&dig)[6],
                                             std::integer_sequence<int, Js...>) {
  constexpr int R = 63 & ~term_mask(6, T);
  int o2 = 0;
#pragma unroll
  for (int q = 2; q < 6; ++q)
    if (R & (1 << q)) o2 += dig[q] * stride_in(R, q, B);
  const double *f2 = sv + std::integral_constant<int, G::ov(T)>::value + o2;
  (tm_st1(tbase + tm_col<RM>(T) + 2 * Js, f2[VOffJ<R, B, RM, Js>::value]), ...);
}
template <class G, int B, int RM, int... Ts>
__device__ __forceinline__ void tm_fill(uint32_t tbase, const double *sv, const int (&dig)[6],
                                        std::integer_sequence<int, Ts...>) {
  ((tm_term(Ts) ? tm_fill_term<G, B, RM, Ts>(tbase, sv, dig, std::make_integer_sequence<int, tm_vcount<RM>(Ts)>{})
                : (void)0),
   ...);
  tm_wait_st();
}
// rows [9 C, 9 C + 9) of a term whose 27 values are the tile rows themselves
template <class G, int B, int RM, int S, int C, int... Is>
__device__ __forceinline__ void tm_rows27(double (&acc)[G::ROWS], const double *f1, uint32_t tcol,
                                          std::integer_sequence<int, Is...>) {
  double v[9];
  tm_ld9(tcol + 18 * C, v);
  ((acc[9 * C + Is] = fma(-f1[RowOff<S, B, RM, 9 * C + Is>::value], v[Is], acc[9 * C + Is])), ...);
}

// ---- consumer: one term on the thread's elements.  dig[q] = the thread's
// index of mode q (modes 1 .. Q0-1) or its group bit (register modes) ----
template <class G, int B, int RM, int T, int... Rs>
__device__ __forceinline__ void term(double (&acc)[G::ROWS], const double *su, const double *sv, const int (&dig)[6],
                                     uint32_t tbase, std::integer_sequence<int, Rs...>) {
  constexpr int S = term_mask(6, T);
  constexpr int R = 63 & ~S;
  if constexpr (G::TM && tm_term(T)) {
    // second factor from the lane's tensor-memory copy
    int o1 = 0;
#pragma unroll
    for (int q = 1; q < 6; ++q)
      if (S & (1 << q)) o1 += dig[q] * stride_in(S, q, B);
    const double *f1 = su + std::integral_constant<int, G::ou(T)>::value + o1;
    const uint32_t tcol = tbase + tm_col<RM>(T);
    if constexpr (tm_vcount<RM>(T) == 9) {
      double v[9];
      tm_ld9(tcol, v);
      ((acc[Rs] = fma(-f1[RowOff<S, B, RM, Rs>::value], v[VJ<R, B, RM, Rs>::value], acc[Rs])), ...);
    } else {
      static_assert(tm_vcount<RM>(T) == 27 && G::ROWS == 27, "27-value terms index the tile rows");
      tm_rows27<G, B, RM, S, 0>(acc, f1, tcol, std::make_integer_sequence<int, 9>{});
      tm_rows27<G, B, RM, S, 1>(acc, f1, tcol, std::make_integer_sequence<int, 9>{});
      tm_rows27<G, B, RM, S, 2>(acc, f1, tcol, std::make_integer_sequence<int, 9>{});
    }
    return;
  }
  int o1 = 0, o2 = 0;
#pragma unroll
  for (int q = 1; q < 6; ++q) {
    if (S & (1 << q)) o1 += dig[q] * stride_in(S, q, B);
    else o2 += dig[q] * stride_in(R, q, B);
  }
  const double *f1 = su + std::integral_constant<int, G::ou(T)>::value + o1;
  const double *f2 = sv + std::integral_constant<int, G::ov(T)>::value + o2;
  BCG_CHECK((o1 >= 0 && o1 + RowOff<S, B, RM, G::ROWS - 1>::value < ipow(B, popc(S) - 1)), "u factor", o1);
  BCG_CHECK((o2 >= 0 && o2 + RowOff<R, B, RM, G::ROWS - 1>::value < ipow(B, 6 - popc(S))), "v factor", o2);
  ((acc[Rs] = fma(-f1[RowOff<S, B, RM, Rs>::value], f2[RowOff<R, B, RM, Rs>::value], acc[Rs])), ...);
}
template <class G, int B, int RM, int... Ts>
__device__ __forceinline__ void terms(double (&acc)[G::ROWS], const double *su, const double *sv, const int (&dig)[6],
                                      uint32_t tbase, std::integer_sequence<int, Ts...>) {
  (term<G, B, RM, Ts>(acc, su, sv, dig, tbase, std::make_integer_sequence<int, G::ROWS>{}), ...);
}
// modes 2..5 of a sub-slab, row-major
template <class G, int B, int RM, int... Rs>
__device__ __forceinline__ void rows_load(double (&acc)[G::ROWS], const double *p, std::integer_sequence<int, Rs...>) {
  ((acc[Rs] = p[RowOff<0x3c, B, RM, Rs>::value]), ...);
}
template <class G, int B, int RM, int... Rs>
__device__ __forceinline__ void rows_store_global(const double (&acc)[G::ROWS], double *p,
                                                  std::integer_sequence<int, Rs...>) {
  (__stcs(p + RowOff<0x3c, B, RM, Rs>::value, acc[Rs]), ...);  // C_6 is written once: streaming stores
}

}  // namespace rs

#ifndef BCG_RS_OPAQUE
#define BCG_RS_OPAQUE 1
#endif
#ifndef BCG_RS_PREFETCH
#define BCG_RS_PREFETCH 6
#endif
constexpr int kPrefetchUnits = BCG_RS_PREFETCH;  // M_6 units prefetched into L2 ahead of the ring

template <int B, int RM, int NGRP, int NU, int XB, int LO, int HINT, int PP, int TM>
__global__ void __launch_bounds__(rs::Geo<B, RM, NGRP, NU, XB, LO, HINT, PP, TM>::NTHREADS, 1)
    k_recursion_stream6(RecFactArgs a) {
  using G = rs::Geo<B, RM, NGRP, NU, XB, LO, HINT, PP, TM>;
  constexpr int NT = G::NT, NS = G::NS;
  extern __shared__ __align__(128) unsigned char rs_smem[];
  double *sv = reinterpret_cast<double *>(rs_smem);
  double *su = sv + G::SEGV;          // [NU][SEGU]
  double *sm = su + G::NU * G::SEGU;  // [NS][UNIT]
  uint64_t *bars = reinterpret_cast<uint64_t *>(sm + NS * G::UNIT);
  uint64_t *mfull = bars, *mempty = bars + G::MF;
  uint64_t *ufull = mempty + NS, *uempty = ufull + G::UF;
  uint64_t *vfull = uempty + G::NU, *vempty = vfull + 1;
  uint64_t *done = vempty + 1;                                  // TM: consumers finished (before the dealloc)
  uint32_t *tslot = reinterpret_cast<uint32_t *>(done + 1);     // TM: allocated tensor-memory base

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < G::MF; ++i) rs::bar_init(&mfull[i], 1);
    for (int i = 0; i < NS; ++i) rs::bar_init(&mempty[i], G::GW);
    for (int i = 0; i < G::UF; ++i) rs::bar_init(&ufull[i], 1);
    for (int i = 0; i < G::NU; ++i) rs::bar_init(&uempty[i], G::UPS * G::GW);
    rs::bar_init(vfull, 1);
    rs::bar_init(vempty, NGRP * G::GW);
    rs::bar_init(done, NGRP * G::GW);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if constexpr (TM) {
    static_assert(!TM || (PP == 1 && rs::tm_cols<RM>() * ((NGRP * G::GW + 3) / 4) <= 512), "tensor-memory columns");
    if (warp == 0) {  // the whole SM's 512 columns (one CTA per SM)
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(rs::su32(tslot))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  }
  __syncthreads();
  uint32_t tbase = 0;
  if constexpr (TM) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    // this warp's lanes (quadrant warp % 4) and its column range among the
    // consumer warps sharing the quadrant
    tbase = *tslot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(rs::tm_cols<RM>() * ((warp - G::PW) >> 2));
    BCG_CHECK((warp < G::PW || ((tbase & 0xffffu) - (*tslot & 0xffffu)) + rs::tm_cols<RM>() <= 512u), "tensor-memory columns",
              tbase & 0xffffu);
  }

  // this CTA's positions [pbeg, pend) of the work list
  const int64_t pbeg = a.nkeys * blockIdx.x / gridDim.x, pend = a.nkeys * (blockIdx.x + 1) / gridDim.x;
  auto item = [&](int64_t pos) -> int64_t { return a.order ? (int64_t)__ldg(a.order + pos) : pos; };
  // V (the 25 second factors) depends on the key's modes 1..5 only: reload
  // it only when one of its block offsets changes
  auto same_v = [&](int64_t it, int64_t prev) -> bool {
    const int32_t *x = a.term_off + it * 2 * NT + 1, *y = a.term_off + prev * 2 * NT + 1;
    bool eq = true;
#pragma unroll
    for (int T = 0; T < NT; ++T) eq = eq && __ldg(x + 2 * T) == __ldg(y + 2 * T);
    return eq;
  };
  auto pwait = [&](uint64_t *b, uint32_t parity) {
    if constexpr (PP == 2) rs::bar_wait_div(b, parity);
    else rs::bar_wait(b, parity);
  };
  if (warp == 0 && (PP != 2 || lane == 31)) {
    // ---- M_6 producer (one lane): units in (position, i0, unit) order into the ring ----
    if (lane == (PP == 2 ? 31 : 0)) {
      int64_t u = 0;
      const uint64_t pol = HINT ? rs::policy_evict_first() : 0;  // M_6 is read once
      static_assert(kPrefetchUnits <= G::UPB, "prefetch at most one block ahead");
      for (int64_t pos = pbeg; pos < pend; ++pos) {
        const double *blk = a.mk + __ldg(a.blk_off + item(pos));
        const double *nblk = pos + 1 < pend ? a.mk + __ldg(a.blk_off + item(pos + 1)) : nullptr;
        if (pos == pbeg)
          for (int j = 0; j < kPrefetchUnits; ++j) rs::bulk_prefetch_l2(blk + (int64_t)j * G::UNIT, 8u * G::UNIT);
        for (int j = 0; j < G::UPB; ++j, ++u) {
          if (kPrefetchUnits > 0) {  // L2 prefetch kPrefetchUnits ahead of the ring
            const int jp = j + kPrefetchUnits;
            if (jp < G::UPB) rs::bulk_prefetch_l2(blk + (int64_t)jp * G::UNIT, 8u * G::UNIT);
            else if (nblk) rs::bulk_prefetch_l2(nblk + (int64_t)(jp - G::UPB) * G::UNIT, 8u * G::UNIT);
          }
          const int st = (int)(u % NS);
          if (u >= NS) pwait(&mempty[st], (uint32_t)((u / NS - 1) & 1));
          uint64_t *fb = &mfull[u % G::MF];
          rs::bar_expect(fb, 8u * G::UNIT);
          if constexpr (HINT) rs::bulk_g2s_hint(sm + (int64_t)st * G::UNIT, blk + (int64_t)j * G::UNIT, 8u * G::UNIT, fb, pol);
          else rs::bulk_g2s(sm + (int64_t)st * G::UNIT, blk + (int64_t)j * G::UNIT, 8u * G::UNIT, fb);
        }
      }
    }
    if constexpr (TM) {  // free the tensor memory once every consumer warp is done with it
      __syncwarp();
      rs::bar_wait(done, 0);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(*tslot) : "memory");
    }
    return;
  }
  if (PP == 2 ? (warp == 0) : (warp == 1 && PP == 1)) {
    if (lane >= NT) return;
    constexpr unsigned kMask = (1u << NT) - 1;
    // ---- factor producer, one lane per term: the 25 copies of a V or U load
    // are ONE warp instruction each (the single-lane version issues 25 bulk
    // copies + 25 offset loads per slab through the same MIO queue the
    // consumers' LDS keep full, and the consumers end up waiting on U) ----
    static_assert(NT <= 32, "one lane per term");
    const bool act = lane < NT;
    const int T = act ? lane : 0;
    const int sS = rs::popc(rs::term_mask(6, T)), rR = 6 - sS;
    const uint32_t vbytes = 8u * rs::ipow(B, rR), ubytes = 8u * rs::ipow(B, sS - 1);
    const int ulen = rs::ipow(B, sS - 1);
    double *vdst = sv + G::ov(T), *udst = su + G::ou(T);
    const double *vsrc = rR <= 3 ? a.cum[rR] : a.cmom[rR];
    const double *usrc = a.cum[sS];
    const uint64_t pol = HINT ? rs::policy_evict_last() : 0;
    int64_t e = -1, s = 0;
    int32_t pv = 0;
    for (int64_t pos = pbeg; pos < pend; ++pos) {
      const int64_t it = item(pos);
      const int32_t *toff = a.term_off + it * 2 * NT;
      const int32_t uo = __ldg(toff + 2 * T), vo = __ldg(toff + 2 * T + 1);
      const bool newv = pos == pbeg || __any_sync(kMask, act && vo != pv);
      pv = vo;
      if (newv) {
        ++e;
        if (e > 0) pwait(vempty, (uint32_t)((e - 1) & 1));
        if (lane == 0) rs::bar_expect(vfull, 8u * G::SEGV);
        __syncwarp(kMask);
        if (act) {
          if constexpr (HINT) rs::bulk_g2s_hint(vdst, vsrc + vo, vbytes, vfull, pol);
          else rs::bulk_g2s(vdst, vsrc + vo, vbytes, vfull);
        }
      }
      for (int i0 = 0; i0 < B; ++i0, ++s) {
        const int buf = (int)(s % G::NU);
        if (s >= G::NU) pwait(&uempty[buf], (uint32_t)((s / G::NU - 1) & 1));
        uint64_t *fb = &ufull[s % G::UF];
        if (lane == 0) rs::bar_expect(fb, 8u * G::SEGU);
        __syncwarp(kMask);
        if (act) {
          if constexpr (HINT) rs::bulk_g2s_hint(udst + buf * G::SEGU, usrc + uo + (int64_t)i0 * ulen, ubytes, fb, pol);
          else rs::bulk_g2s(udst + buf * G::SEGU, usrc + uo + (int64_t)i0 * ulen, ubytes, fb);
        }
      }
    }
    return;
  }
  if (warp == 1 && PP == 0) {
    // ---- factor producer: V per run of equal tails, U per slab ----
    if (lane == 0) {
      int64_t e = -1, s = 0, prev = -1;
      const uint64_t pol = HINT ? rs::policy_evict_last() : 0;  // the factors are re-read by every block sharing them
      for (int64_t pos = pbeg; pos < pend; ++pos) {
        const int64_t it = item(pos);
        const int32_t *toff = a.term_off + it * 2 * NT;
        if (prev < 0 || !same_v(it, prev)) {
          ++e;
          if (e > 0) rs::bar_wait(vempty, (uint32_t)((e - 1) & 1));
          rs::bar_expect(vfull, 8u * G::SEGV);
          rs::load_v_all<G>(sv, a, toff, vfull, pol, std::make_integer_sequence<int, NT>{});
        }
        prev = it;
        for (int i0 = 0; i0 < B; ++i0, ++s) {
          const int buf = (int)(s % G::NU);
          if (s >= G::NU) rs::bar_wait(&uempty[buf], (uint32_t)((s / G::NU - 1) & 1));
          uint64_t *fb = &ufull[s % G::UF];
          rs::bar_expect(fb, 8u * G::SEGU);
          rs::load_u_all<G>(su + buf * G::SEGU, a, toff, i0, fb, pol, std::make_integer_sequence<int, NT>{});
        }
      }
    }
    return;
  }
  // ---- consumers: group grp takes the units u == grp (mod NGRP) ----
  const int ct = threadIdx.x - 32 * G::PW;
  const int grp = ct / G::GT, t = ct % G::GT;
  // lane order (fastest first): the register modes' group bits (last mode
  // fastest), the thread-level modes, then the sub-slab h (measured faster
  // than h-before-thread-modes at cfg5)
  int h = t / G::TPS;
  const int r = t % G::TPS;
  int dig[6];
  dig[0] = 0;
  if constexpr (LO == 1) {
    // lane order chosen with the measured wavefront rule (an LDS.64 costs
    // max(bank rule, ceil(distinct addresses per lane quad / 2)) wavefronts,
    // tools/rs_wavefront_model.py): lane bits 0, 1 = the low bit of the
    // mode-2 digit and the sub-slab, so a quad of lanes reads <= 2 distinct
    // doubles of every factor not holding modes 1 and 2 together; bits 2..4
    // = the group bits of modes 5, 4, 3; the warp = the high part of the
    // mode-2 digit.  0.476 factor wavefronts per element instead of 0.633.
    static_assert(LO != 1 || (RM == 0x38 && B == 6), "lane order 1 is laid out for register modes 3,4,5 at b = 6");
    dig[2] = (t & 1) + 2 * (t >> 5);
    h = (t >> 1) & 1;
    dig[5] = (t >> 2) & 1;
    dig[4] = (t >> 3) & 1;
    dig[3] = (t >> 4) & 1;
  } else {
    int gb = r % (1 << G::NRM), tm = r >> G::NRM;
#pragma unroll
    for (int q = 5; q >= 2; --q) {
      if (RM & (1 << q)) {
        dig[q] = gb & 1;  // group bit of register mode q (index = 2 d + g)
        gb >>= 1;
      } else {
        dig[q] = tm % B;  // thread-level mode
        tm /= B;
      }
    }
  }
  int ebase = 0;  // thread's first element inside its sub-slab (row-major over modes 2..5)
#pragma unroll
  for (int q = 2; q < 6; ++q) ebase += dig[q] * rs::ipow(B, 5 - q);
  int64_t e = -1, s = 0, efill = -1;
  // Per-block information (work item -> M_6 offset, "the second factors
  // change here") is fetched one block AHEAD: the dependent global loads
  // (work list -> block offset, ~2 x L2 latency) held 5% of the consumers'
  // stall samples when issued at the top of the block they are for.  With the
  // host's per-position flags (a.newv, the tail-ordered list) a block costs
  // three loads; without them (a sub-range in list order) the 25 factor
  // offsets of neighbouring blocks are compared as before.
  int64_t it_cur = pbeg < pend ? item(pbeg) : 0;
  int64_t boff_cur = pbeg < pend ? __ldg(a.blk_off + it_cur) : 0;
  bool newv_cur = true;
  for (int64_t pos = pbeg; pos < pend; ++pos) {
    const int64_t it = it_cur, boff = boff_cur;
    const bool newv = newv_cur;
    if (pos + 1 < pend) {  // issue the next block's loads now, use them next iteration
      it_cur = item(pos + 1);
      boff_cur = __ldg(a.blk_off + it_cur);
      newv_cur = a.newv ? __ldg(a.newv + pos + 1) != 0 : !same_v(it_cur, it);
    }
    if (newv) {
      if (e >= 0 && lane == 0) rs::bar_arrive(vempty);  // done with the previous V
      ++e;
    }
    rs::bar_wait(vfull, (uint32_t)(e & 1));
    if constexpr (TM) {
      if (e != efill) {  // new tail: this thread's tail-constant second factors -> its tensor-memory lane
        rs::tm_fill<G, B, RM>(tbase, sv, dig, std::make_integer_sequence<int, NT>{});
        efill = e;
      }
    }
    double *blk = a.mk + boff;
    for (int i0 = 0; i0 < B; ++i0, ++s) {
      const int ub = (int)(s % G::NU);
      for (int p = 0; p < G::UPS; ++p) {
        const int j = i0 * G::UPS + p;
        const int64_t u = (pos - pbeg) * G::UPB + j;
        if ((int)(u % NGRP) != grp) continue;
        const int st = (int)(u % NS);
        dig[1] = G::U1 * p + h;
        rs::bar_wait(&mfull[u % G::MF], (uint32_t)((u / G::MF) & 1));
        double acc[G::ROWS];
        BCG_CHECK((h * G::SUB + ebase + rs::RowOff<0x3c, B, RM, G::ROWS - 1>::value < G::UNIT), "element", ebase);
        rs::rows_load<G, B, RM>(acc, sm + (int64_t)st * G::UNIT + h * G::SUB + ebase,
                                 std::make_integer_sequence<int, G::ROWS>{});
        // the LDS above are only issued, not necessarily performed: order them
        // before the bulk-copy engine's refill of this stage (async proxy)
        // that the arrive below allows -- without this fence the refill can
        // land first (seen as 76-224 corrupted elements of one block per
        // launch when the producer already waits on this very stage)
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) rs::bar_arrive(&mempty[st]);  // refill the stage
        rs::bar_wait(&ufull[s % G::UF], (uint32_t)((s / G::UF) & 1));
#if BCG_RS_OPAQUE
        // keep the 50 per-term factor offsets out of registers: without this
        // the compiler hoists them out of the unit loop (loop-invariant),
        // which costs ~50 registers per thread and with them a consumer group
#pragma unroll
        for (int q = 1; q < 6; ++q) asm volatile("" : "+r"(dig[q]));
#endif
        rs::terms<G, B, RM>(acc, su + ub * G::SEGU, sv, dig, tbase, std::make_integer_sequence<int, NT>{});
        __syncwarp();
        if (lane == 0) rs::bar_arrive(&uempty[ub]);
        rs::rows_store_global<G, B, RM>(acc, blk + (int64_t)j * G::UNIT + h * G::SUB + ebase,
                                         std::make_integer_sequence<int, G::ROWS>{});
      }
    }
  }
  if (e >= 0 && lane == 0) rs::bar_arrive(vempty);
  if constexpr (TM) {
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncwarp();
    if (lane == 0) rs::bar_arrive(done);
  }
}

// variant choice (A/B knob BCG_RS_TILE), cfg5 layout, L2 flushed, same box
// (profiles/r02_recursion_stream.txt; every variant bitwise equal to v2):
//   default (v9): v8 + the 81 tail-constant second-factor values of a thread
//      cached in its tensor-memory lane (tcgen05.st per tail, tcgen05.ld per
//      unit instead of 81 of 391 shared-memory loads)              10.68 ms (v8 on that box: 11.21)
//   16 (v8): register modes 3,4,5 (27 elements), 4 consumer groups (12
//      warps, 128 registers), quad-aware lane order, 4 U buffers + 3 ring
//      stages, one producer lane per term, L2 eviction hints      10.89 ms
//   0: v7d -- lane order g5,g4,g3,mode 2,h; 3 U buffers + 4 stages; one
//      lane issues all factor copies; no hints                    11.46 ms
//   1: v7d with 3 consumer groups (165 registers)
//   4: register modes 2..5 (81 elements), 6 consumer warps, 254 registers
//   5: v7d + the lane order          6: 5 + 4 U buffers
//   14: 6 + per-term producer lanes (= v8 without the hints)      11.16 ms
//   17: v8 with ONE producer warp (lane 31 streams M_6, lanes 0..24 the factors) 10.71 ms
//   18: 17 with 5 consumer groups (15 warps, 3 U buffers + 4 stages)   10.80 ms
template <int B, int RM, int NGRP, int NU, int LO = 0, int HINT = 0, int PP = 0, int TM = 0, int XB = 1>
static cudaError_t go_stream6(const RecFactArgs &a, int nsm, cudaStream_t stream) {
  using G = rs::Geo<B, RM, NGRP, NU, XB, LO, HINT, PP, TM>;
  static_assert(G::ok, "stream6 geometry");
  auto kern = k_recursion_stream6<B, RM, NGRP, NU, XB, LO, HINT, PP, TM>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM);
  if (e != cudaSuccess) return e;
  const int64_t grid = a.nkeys < nsm ? a.nkeys : nsm;
  kern<<<(unsigned)grid, G::NTHREADS, G::SMEM, stream>>>(a);
  g_launches++;
  return cudaGetLastError();
}

bool recursion_stream6_supported(int b) { return b == 6; }

cudaError_t launch_recursion_stream6(const RecFactArgs &a, int b, cudaStream_t stream) {
  if (a.nkeys <= 0) return cudaSuccess;
  if (b != 6) return cudaErrorInvalidValue;
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = 148;
  }
  static const int tile = getenv("BCG_RS_TILE") ? atoi(getenv("BCG_RS_TILE")) : -1;
  if (tile == 0) return go_stream6<6, 0x38, 4, 3>(a, nsm, stream);
  if (tile == 1) return go_stream6<6, 0x38, 3, 3>(a, nsm, stream);
  if (tile == 4) return go_stream6<6, 0x3c, 6, 3>(a, nsm, stream);
  if (tile == 5) return go_stream6<6, 0x38, 4, 3, 1>(a, nsm, stream);
  if (tile == 6) return go_stream6<6, 0x38, 4, 4, 1>(a, nsm, stream);
  if (tile == 14) return go_stream6<6, 0x38, 4, 4, 1, 0, 1>(a, nsm, stream);
  if (tile == 16) return go_stream6<6, 0x38, 4, 4, 1, 1, 1>(a, nsm, stream);
  if (tile == 17) return go_stream6<6, 0x38, 4, 4, 1, 1, 2>(a, nsm, stream);
  if (tile == 18) return go_stream6<6, 0x38, 5, 3, 1, 1, 2>(a, nsm, stream);
  return go_stream6<6, 0x38, 4, 4, 1, 1, 1, 1>(a, nsm, stream);
}

}  // namespace bcg
