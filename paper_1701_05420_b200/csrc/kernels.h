// Kernel launch interfaces shared by the C ABI (capi.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "plan.h"

namespace bcg {

struct MomentArgs {
  const double *x;
  int64_t t, ldx;
  int n, h, r;
  int bulk_ok;  // rows contiguous and 16-byte aligned: TMA bulk staging
  // x is the TRANSPOSED data (n rows, row stride ldx >= padded_t(t)), zero-padded past t
  const int16_t *rowcols, *colcols;
  const int32_t *row_keybase, *row_olin, *row_cstart;
  const int32_t *col_rank, *col_olin, *col_size;
  const int64_t *offs;  // per GEMM key: output offset of its block, -1 = not produced
  const Tile *tiles;
  const int32_t *tile_kmin, *tile_kmax;
  int ntiles;
  int64_t R, C;
  int nslices;        // slices in this launch (group)
  int slice0;         // first slice of the group
  int nslices_total;  // slices over the whole sample range
  int64_t slice_len;
  double *out, *ws;
  int64_t S;
  int32_t kmin_sel, kmax_sel;
};

// fixed split-K slice length (samples): the summation order of every element
// depends on t only (see moment.cu).  Longer slices cut the partials' DRAM
// traffic but cost wave balance (profiles/r02_moment_experiments.log (7)).
#ifndef BCG_SLICE_LEN
#define BCG_SLICE_LEN 16384
#endif
constexpr int64_t kSliceLen = BCG_SLICE_LEN;
size_t moment_smem_bytes(int KC, int n, int tm = 64, int tn = 64);
int pick_kc(int n);
bool v1_shape_supported(int KC, int m, int tm, int tn);
cudaError_t launch_moment(const MomentArgs &args, int KC, int grid, cudaStream_t stream, int tm = 64, int tn = 64);
cudaError_t launch_reduce_slices(const double *ws, int nslices, int64_t S, int64_t lo, int64_t hi,
                                 double *out, cudaStream_t stream);

cudaError_t launch_colstats(const double *x, int64_t t, int64_t n, int64_t ldx, double *sums, double *mean,
                            double *sumsq, int64_t *first_bad, double *scratch, int nparts,
                            cudaStream_t stream);
int colstats_parts(int64_t t, int64_t n);
cudaError_t launch_center(const double *x, int64_t t, int64_t n, int64_t ldx, const double *mean, double *xc,
                          cudaStream_t stream);
cudaError_t launch_transpose(const double *xt, int64_t n, int64_t t, double *x, cudaStream_t stream);
cudaError_t launch_transpose_pad(const double *x, int64_t t, int64_t n, int64_t ldx, const double *mean, double *xt,
                                 int64_t ldt, cudaStream_t stream);
cudaError_t launch_pad_rows(const double *src, int64_t n, int64_t t, int64_t lds, double *dst, int64_t ldt,
                            cudaStream_t stream);
cudaError_t launch_rowstats(const double *xt, int64_t n, int64_t t, int64_t ldt, double *sums, double *sumsq,
                            double *ws, int P, cudaStream_t stream);
int rowstats_parts(int64_t n, int64_t t);
// Staging of a chunk's n variables by 2-D TMA boxes of <= 256 rows: n <= 256
// is one box of exactly n rows; wider data takes ceil(n / 256) boxes of equal
// height (a multiple of 8 rows, so every box starts 1024-byte aligned for the
// 128-byte swizzle).
__host__ __device__ inline int xbox_count(int n) { return (n + 255) / 256; }
__host__ __device__ inline int xbox_rows(int n) {
  if (n <= 256) return n;
  const int nb = xbox_count(n);
  return ((n + nb - 1) / nb + 7) / 8 * 8;
}
__host__ __device__ inline int xstaged_rows(int n) { return xbox_count(n) * xbox_rows(n); }

// padded sample count of the transposed layout the moment kernel reads
inline int64_t padded_t(int64_t t) { return (t + 15) / 16 * 16; }
cudaError_t launch_sym_fill(const int32_t *fill_keys, int64_t nfill, const int32_t *keys, const int64_t *offs, int m,
                            int b, int64_t n, double *out, cudaStream_t stream);
cudaError_t launch_div(int64_t len, const double *x, double d, double *out, cudaStream_t stream);
cudaError_t launch_axpby(int64_t len, double a, const double *x, double c, const double *y, double *out,
                         cudaStream_t stream);

struct RecursionArgs {
  int m, b;
  int64_t n;
  int64_t K;
  const int64_t *offs;
  const int32_t *keys;      // K x m, 1-based
  const int32_t *sub_rank;  // K x nslots
  const int32_t *part_mask; // per partition 8 masks
  int nslots;
  int p_begin, p_end;       // partitions [p_begin, p_end) processed
  int64_t k0, k1;           // output blocks [k0, k1) processed
  const int32_t *klist;     // if non-null: process klist[0 .. k1-k0) instead of the range
  int sigma_lo, sigma_hi;   // sigma range (for grouping into B_sigma)
  int sigma_first[12];       // sigma -> first partition (host copy)
  const int64_t *lower_offs[16];
  const double *lower[16];  // index = order
  double *mk;               // in/out
  int mode;                 // 0: mk = mk - sum_sigma B_sigma ; 1: mk = B_sigma (single sigma)
  int64_t e0, e1;           // only elements mk[e0 .. e1) are written (element-span split)
};
cudaError_t launch_recursion(const RecursionArgs &args, cudaStream_t stream);

struct RecFactArgs {
  int64_t nkeys;            // full output blocks to process (work items 0 .. nkeys-1)
  const int64_t *blk_off;   // [nkeys] M_m element offset of each block
  const int32_t *term_off;  // [nkeys][nterms][2] element offsets of each term's factor blocks
  const double *cum[16];    // packed C_k, k = 2 .. m-2
  const double *cmom[16];   // packed central moments M_k, k = 4 .. m-2
  double *mk;               // in: M_m, out: C_m
  const int32_t *order;     // v7 only: position -> work item (null: identity)
  const int32_t *newv;      // v7 only: per position, 1 = second factors differ from the previous position's (null: compare)
};
int recursion_fact_terms(int m);
bool recursion_fact_supported(int m, int b);
cudaError_t launch_recursion_fact(const RecFactArgs &a, int m, int b, cudaStream_t stream);
// v7 (recursion_stream.cu): order 6, b = 6, every pointer 16-byte aligned
bool recursion_stream6_supported(int b);
cudaError_t launch_recursion_stream6(const RecFactArgs &a, int b, cudaStream_t stream);

// dense-entry verification (dense.cu)
int dense_subsets_parts(int64_t E, int64_t t);
cudaError_t launch_dense_subsets(const double *x, int64_t t, int64_t n, int64_t ldx, const double *mean, int m,
                                 const int32_t *idx, int64_t E, double *part, int P, double *out,
                                 cudaStream_t stream);

extern int64_t g_launches;

}  // namespace bcg
