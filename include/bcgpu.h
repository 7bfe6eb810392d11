/*
 * bcgpu -- B200-native (sm_100a) moment / cumulant engine, C ABI.
 *
 * Drop-in boundary for the reference package `blockcumulants`
 * (/root/reference/pkg/src/blockcumulants, cited as bc/<file>:<line>).  The
 * reference's only native boundary is the Cython module `_core`
 * (bc/_core.pyx:126-175, imported at bc/_engines.py:26-31); everything the
 * Python layer above it needs on the hot path -- centering, packed moments,
 * the cumulant recursion -- is exported here with plain pointers and sizes.
 *
 * Conventions
 *  - Every device pointer is caller-owned device memory (torch allocations in
 *    the Python host layer).  Plans own only their small index tables.
 *  - Every call is stream-ordered on `stream` (a cudaStream_t, passed as void*;
 *    NULL = legacy default stream) and returns a status code; on failure
 *    bcg_last_error() describes it (thread-local).
 *  - Status codes map to the reference's error convention (bc/errors.py:4-9):
 *    BCG_EINVAL -> ValidationError, BCG_ENOMEM -> MemoryError,
 *    BCG_ECUDA -> RuntimeError.
 *  - Packed tensors use the reference's flat layout exactly: block k (k-th
 *    sorted key in lexicographic order, bc/symtensor.py:47-49) occupies
 *    [offs[k], offs[k+1]) row-major over its edges (bc/_engines.py:46-61).
 *  - All values are float64, all index tables int64 (C `long` on Linux, as the
 *    reference's memoryviews require, bc/_core.pyx:126-128).
 */
#ifndef BCGPU_H
#define BCGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BCG_OK 0
#define BCG_EINVAL 1
#define BCG_ECUDA 2
#define BCG_ENOMEM 3

/* Last error message of the calling thread ("" if none). */
const char *bcg_last_error(void);
/* ABI version (major*100 + minor). */
int bcg_version(void);
/* Number of kernel launches this library has issued in this process
 * (evidence counter for bench.py's `gpu_launches`). */
int64_t bcg_launch_count(void);

/* ---------------------------------------------------------------------------
 * Drop-in replacement for `_core.moment_blocks` (bc/_core.pyx:126-148).
 * Same arguments and semantics, on DEVICE pointers:
 *   out[offs[k] + rowmajor(o)] += sum_l prod_q xt[(col0[k,q] + o_q) * t + l]
 * for blocks k in [k0, k1); raw product sums ACCUMULATED (no 1/t, caller
 * zero-fills and scales, bc/_engines.py:92-100).  xt is (n, t) row-major as the
 * reference passes it (bc/_engines.py:95); col0/edges are (K, m) int64, offs is
 * (K+1) int64.  Errors as the reference: m outside [2, 16] -> BCG_EINVAL
 * ("kernel supports 2 <= m <= 16", bc/_core.pyx:138-139).  Deterministic:
 * repeated calls produce bitwise-identical sums.  The layout passed in must
 * be the reference's (_block_layout of some (n, m, b)); it is checked.
 * ------------------------------------------------------------------------- */
int bcg_moment_blocks(const double *xt, int64_t n, int64_t t,
                      const int64_t *col0, const int64_t *edges, int64_t m,
                      int64_t K, double *out, const int64_t *offs, int64_t k0,
                      int64_t k1, void *stream);

/* ---------------------------------------------------------------------------
 * Plans: host-built (C++) index tables for one (n, m, b), uploaded once.
 * A plan for order m serves the order-m moment GEMM (bc/_engines.py:83-100)
 * and the order-m cumulant recursion (bc/cumulants.py:53-136).
 * ------------------------------------------------------------------------- */
typedef struct bcg_plan bcg_plan;

/* Symmetric plan (the default): inside a block whose key repeats a block
 * index j (e.g. key (1,1,2,...)), the elements whose in-block digits differ
 * only by a permutation within that run are equal (the moment tensor is
 * super-symmetric).  The moment GEMM then produces only the elements whose
 * digits are non-decreasing within the runs of its row / column tuple and a
 * fill pass copies the sorted element to its permutations (K2):
 * 58% of the stored elements at order 6 (cfg4, cfg5), 70% at order 4 (cfg2).
 * Every stored element is still written; accumulate semantics hold for an
 * `out` that is already symmetric within blocks (e.g. zero).  The reference
 * computes every stored element directly (bc/_core.pyx:60-123); values agree
 * to rounding (the permuted products are formed in another order). */
int bcg_plan_create(int64_t n, int32_t m, int32_t b, bcg_plan **plan);
/* Same with an explicit moment-kernel variant (-1 = default, 0 = the DMMA
 * kernel of DESIGN.md K2; other values are rejected). */
int bcg_plan_create_ex(int64_t n, int32_t m, int32_t b, int32_t variant,
                       bcg_plan **plan);
/* Plan flags: BCG_PLAN_FULL -- the moment GEMM produces every stored element
 * directly, element-wise accumulate semantics for any prior `out` (what the
 * drop-in bcg_moment_blocks uses); BCG_PLAN_HOST -- tables only, nothing
 * uploaded (layout queries / selfcheck without a GPU). */
#define BCG_PLAN_FULL 1
#define BCG_PLAN_HOST 2
int bcg_plan_create_flags(int64_t n, int32_t m, int32_t b, int32_t flags,
                          bcg_plan **plan);
/* Moment-kernel choice of the plan: variant (0 = v1), CTA tile tm x tn of
 * its first GEMM (picked per GEMM by the staircase tile model) and the number
 * of tiles over all its GEMMs. */
int bcg_plan_kernel(const bcg_plan *plan, int32_t *variant, int32_t *tm,
                    int32_t *tn, int64_t *ntiles);
/* The plan's moment GEMMs: 1, or 2 for a hybrid odd-order plan (keys split
 * by their middle entry at split_T: key[h] >= T -> an (h | m-h) GEMM, else
 * (h+1 | m-h-1)).  Gemm i (< *ngemm) is described by info[0..3] = h, r, tm,
 * tn and *ntiles; pass i < 0 to query only *ngemm and *split_T. */
int bcg_plan_gemm(const bcg_plan *plan, int32_t i, int32_t *ngemm, int32_t *split_T,
                  int32_t *info, int64_t *ntiles);
/* Output size of bcg_moment_raw on this plan (S_m) and the number of
 * elements its GEMMs compute (S_m for a full plan, fewer for a symmetric one:
 * 2 * t * produced is the FP64 work the DMMA kernel executes). */
int bcg_plan_output(const bcg_plan *plan, int64_t *S_out, int64_t *produced);
/* Elements the moment GEMMs' CTA tiles cover (tiled area incl. masked
 * staircase and edge positions; produced / tiled is the tile efficiency) and
 * the number of narrow band-edge tiles among them. */
int bcg_plan_tiled(const bcg_plan *plan, int64_t *tiled, int64_t *edge_tiles);
/* Waste breakdown of the staircase cover (introspection, tools/tile_waste.py):
 * out[0] tiled area, out[1] valid pairs, out[2] area of empty 8 x 8 sub-tiles,
 * out[3] area of empty 32 x 32 warp tiles, out[4] overhang past R / C. */
int bcg_plan_waste(const bcg_plan *plan, int64_t *out);
/* Host-only plan (tables built, nothing uploaded): layout queries work
 * without a GPU; compute calls on it fail with BCG_EINVAL. */
int bcg_plan_create_host(int64_t n, int32_t m, int32_t b, bcg_plan **plan);
int bcg_plan_destroy(bcg_plan *plan);
/* Host-side verification of the moment GEMM mapping: every element the GEMMs
 * produce comes from exactly one (tile, row, col) and reads exactly the data
 * columns of its (key, offsets); every stored element is produced or (symmetric
 * plan) is a within-run permutation of a produced one in a fill-listed block.
 * BCG_OK or BCG_EINVAL with a message. */
int bcg_plan_selfcheck(const bcg_plan *plan);
/* K = number of stored blocks, S = stored elements (offs[K]) of order `order`
 * (1 <= order <= m). */
int bcg_plan_sizes(const bcg_plan *plan, int32_t order, int64_t *K, int64_t *S);
/* Copy the reference layout of order `order` (keys 1-based, col0, edges: K x
 * order; offs: K+1) into caller HOST buffers (bc/_engines.py:46-54). */
int bcg_plan_layout(const bcg_plan *plan, int32_t order, int64_t *keys,
                    int64_t *col0, int64_t *edges, int64_t *offs);
/* Workspace bytes bcg_moment_raw(_range) needs for t samples (0 = none):
 * the transposed copy of x plus the split-K partials. */
int bcg_moment_ws_bytes(const bcg_plan *plan, int64_t t, size_t *bytes);
/* Workspace bytes of the transposed-input entries bcg_moment_raw_t(_range):
 * the split-K partials only. */
int bcg_moment_t_ws_bytes(const bcg_plan *plan, int64_t t, size_t *bytes);

/* ---------------------------------------------------------------------------
 * Column statistics of x (t x n row-major, leading dimension ldx >= n):
 * sums[n] (if non-NULL) = sum_l x[l, c]; mean[n] (if non-NULL) = sums / t
 * (bc/moments.py:41); sumsq[n] (if non-NULL) = sum_l x[l, c]^2;
 * first_bad (if non-NULL, device int64) = smallest row-major linear index of a
 * non-finite element or -1 -- the reference's isfinite scan and its "row r,
 * column c" diagnostic (bc/moments.py:23-35).  Deterministic reduction order.
 * ------------------------------------------------------------------------- */
int bcg_colstats(const double *x, int64_t t, int64_t n, int64_t ldx,
                 double *sums, double *mean, double *sumsq, int64_t *first_bad,
                 void *ws, size_t ws_bytes, void *stream);
/* Workspace bytes bcg_colstats needs (per-partition partial sums). */
size_t bcg_colstats_ws_bytes(int64_t t, int64_t n);

/* xc[l, c] = x[l, c] - mean[c]   (bc/moments.py:38-41). */
int bcg_center(const double *x, int64_t t, int64_t n, int64_t ldx,
               const double *mean, double *xc, void *stream);

/* ---------------------------------------------------------------------------
 * Order-m packed RAW moment sums of x (t x n row-major, ldx >= n), ACCUMULATED
 * into out[S_m] (same semantics as bcg_moment_blocks over all blocks).  The
 * Khatri-Rao-staged FP64 DMMA GEMM; x is first transposed
 * into the workspace.  `ws` must hold bcg_moment_ws_bytes(plan, t) bytes.
 * ------------------------------------------------------------------------- */
int bcg_moment_raw(const bcg_plan *plan, const double *x, int64_t t,
                   int64_t ldx, double *out, void *ws, size_t ws_bytes,
                   void *stream);
/* Same from the TRANSPOSED layout the reference's own kernel takes
 * (bc/_engines.py:95): xt has n rows of stride ldt (even, >= bcg_padded_t(t)),
 * 16-byte aligned, zero-padded in [t, ldt).  No transpose pass; `ws` needs
 * bcg_moment_t_ws_bytes(plan, t) bytes (the split-K partials). */
int bcg_moment_raw_t(const bcg_plan *plan, const double *xt, int64_t t,
                     int64_t ldt, double *out, void *ws, size_t ws_bytes,
                     void *stream);
/* t rounded up to the moment kernel's 16-sample chunk. */
int64_t bcg_padded_t(int64_t t);
/* xt[c, l] = x[l, c] - mean[c] (mean may be NULL) for l < t, 0 for
 * t <= l < ldt: centering (bc/moments.py:38-41) fused with the transpose
 * into the layout bcg_moment_raw_t reads. */
int bcg_transpose_pad(const double *x, int64_t t, int64_t n, int64_t ldx,
                      const double *mean, double *xt, int64_t ldt, void *stream);
/* Per-row sums / sums of squares of xt (n x ldt, first t entries): the
 * column statistics of the transposed data (_check_centered,
 * bc/cumulants.py:31-39).  Deterministic. */
int bcg_rowstats(const double *xt, int64_t n, int64_t t, int64_t ldt,
                 double *sums, double *sumsq, void *stream);
/* Same, split into row segments so small n still fills the GPU; `ws` must
 * hold bcg_rowstats_ws_bytes(n, t) bytes (segment partials, added in segment
 * order: deterministic). */
size_t bcg_rowstats_ws_bytes(int64_t n, int64_t t);
int bcg_rowstats_ws(const double *xt, int64_t n, int64_t t, int64_t ldt,
                    double *sums, double *sumsq, void *ws, size_t ws_bytes,
                    void *stream);
/* Same, restricted to blocks [k0, k1) (only out[offs[k0]:offs[k1]] is
 * touched; bitwise identical to the full call on those blocks) -- the
 * block-split path of moment_parallel_blocks (bc/moments.py:99-131). */
int bcg_moment_raw_range(const bcg_plan *plan, const double *x, int64_t t,
                         int64_t ldx, double *out, void *ws, size_t ws_bytes,
                         int64_t k0, int64_t k1, void *stream);
/* bcg_moment_raw_t restricted to blocks [k0, k1): the per-rank moment of the
 * block-split multi-GPU mode (distributed.cumulants_upto_block_split), every
 * rank reading all of xt; bitwise identical to the full call on its blocks. */
int bcg_moment_raw_t_range(const bcg_plan *plan, const double *xt, int64_t t,
                           int64_t ldt, double *out, void *ws, size_t ws_bytes,
                           int64_t k0, int64_t k1, void *stream);

/* ---------------------------------------------------------------------------
 * Cumulant recursion, in place: on entry mk holds the order-m central moment
 * M_m (packed, order of `plan`), on exit C_m = (M_m - B_2) - B_3 - ... with
 *   B_sigma[key][o] = sum over min-2 partitions zeta of (1..m) into sigma
 *                     parts (bc/partitions.py:63-98 order) of
 *                     prod_{part} C_|part|[key|part][o|part]
 * (bc/cumulants.py:53-84, 119-136).  lower[j] = packed C_{j+2} (device), for
 * j = 0 .. m-4.  m <= 3 is a no-op (the cumulant is the moment).
 * ------------------------------------------------------------------------- */
int bcg_cumulant_recursion(const bcg_plan *plan, double *mk,
                           const double *const *lower, void *stream);

/* Same, for output blocks [k0, k1) only: the block-list split of the
 * recursion across GPUs (north_star; bc/moments.py:114-131 splits the same
 * way across threads).  Only mk[offs[k0]:offs[k1]] is written. */
int bcg_cumulant_recursion_range(const bcg_plan *plan, double *mk,
                                 const double *const *lower, int64_t k0,
                                 int64_t k1, void *stream);

/* Same, with the central moments of the complements: cmom[j] = packed
 * central moment M_{j+2} (device) for j = 2 .. m-4 (orders 4 .. m-2; entries
 * for orders 2, 3 are ignored: M_2 = C_2, M_3 = C_3).  Full blocks then use
 * the factored, register-blocked kernel
 *   C_m = M_m - sum_{S containing mode 1, 2 <= |S| <= m-2} C_|S|[S] M_{m-|S|}[rest]
 * (algebraically the reference's partition sum grouped by the part holding
 * mode 1; 25 products per element at m = 6 instead of 55), for 4 <= m <= 6
 * and b <= 8; other blocks / orders fall back to the partition kernel.  Only
 * blocks [k0, k1) are written.  bcg_cumulant_recursion(_range) use the
 * factored kernel for m <= 5 (no central moments needed). */
int bcg_cumulant_recursion_ex(const bcg_plan *plan, double *mk,
                              const double *const *lower,
                              const double *const *cmom, int64_t k0,
                              int64_t k1, void *stream);

/* Same, for the ELEMENTS mk[e0, e1) only (everything else untouched): the
 * element-balanced split of the top orders across GPUs, where each rank holds
 * the fully reduced M_m on an equal-size span of the packed buffer (an
 * in-place NCCL reduce-scatter) -- the per-element recursion needs nothing
 * else.  Blocks inside the span take the bcg_cumulant_recursion_ex kernels;
 * the at most two blocks the span cuts take the partition kernel with
 * writes masked to the span. */
int bcg_cumulant_recursion_span(const bcg_plan *plan, double *mk,
                                const double *const *lower,
                                const double *const *cmom, int64_t e0,
                                int64_t e1, void *stream);

/* Same correction without the moment: out = B_sigma (bc/cumulants.py:53-84,
 * `outer_prod_cum(m, sigma, lower)`), out has S_m elements. */
int bcg_outer_prod_cum(const bcg_plan *plan, int32_t sigma,
                       const double *const *lower, double *out, void *stream);

/* ---------------------------------------------------------------------------
 * Packed-buffer elementwise ops (BlockSymTensor `+ - scale`,
 * bc/symtensor.py:185-200; the weighted reduction of moment_parallel,
 * bc/moments.py:93-95):  out[i] = a * x[i] + c * y[i]  (y may be NULL -> c
 * ignored).  out may alias x or y.
 * ------------------------------------------------------------------------- */
int bcg_axpby(int64_t len, double a, const double *x, double c,
              const double *y, double *out, void *stream);
/* out[i] = x[i] / d  (the reference's `out /= t`, bc/_engines.py:99). */
int bcg_div(int64_t len, const double *x, double d, double *out, void *stream);

/* ---------------------------------------------------------------------------
 * Dense-entry verification (SURVEY §8 f row 4; the reference's dense oracle
 * bc/oracle.py:89-117 is limited to n^m <= 1e8): for E element tuples
 * idx[E][m] (0-based column indices, any order, repeats allowed) of the
 * row-major data x (t rows, row stride ldx >= n, device) with column means
 * mean[n], out[e][S] = sum_l prod_{q in S} (x[l, idx[e][q]] - mean[idx[e][q]])
 * for every subset S of {0..m-1} (bit q of S = index q; out[e][0] = t),
 * 1 <= m <= 8.  Independent of the block layout and of the moment / recursion
 * kernels; deterministic.  Workspace: bcg_dense_subsets_ws_bytes(E, m, t)
 * bytes.
 * ------------------------------------------------------------------------- */
size_t bcg_dense_subsets_ws_bytes(int64_t E, int32_t m, int64_t t);
int bcg_dense_subsets(const double *x, int64_t t, int64_t n, int64_t ldx,
                      const double *mean, int32_t m, const int32_t *idx,
                      int64_t E, double *out, void *ws, size_t ws_bytes,
                      void *stream);

#ifdef __cplusplus
}
#endif

#endif /* BCGPU_H */
