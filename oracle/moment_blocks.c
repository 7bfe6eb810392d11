/*
 * ORACLE -- test infrastructure only (tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may call it, as the CHECKER; the product path
 * never does).  Plain-C restatement of the reference's native moment kernel.
 *
 * Restates /root/reference/pkg/src/blockcumulants/_core.pyx:126-148
 * (`moment_blocks`) and its per-block worker `_one_block` (_core.pyx:60-123):
 *
 *   for every block k in [k0, k1):
 *     for every within-block offset tuple o (row-major over edges[k][:]):
 *       out[offs[k] + rowmajor(o)] += sum_l prod_q xt[col0[k][q] + o_q][l]
 *
 * i.e. RAW product sums, ACCUMULATED into `out` (no 1/t; the caller zero-fills
 * and scales, _engines.py:92-100).  `xt` is the transposed (n, t) data, one
 * contiguous row per variable, as the reference passes it (_engines.py:95).
 *
 * The summation order differs from the reference (which keeps four-lane
 * partials over 512-sample chunks, _core.pyx:18-30, 80-83): here a prefix
 * product over the first m-1 modes is formed per sample chunk and the last
 * mode is a plain sequential dot product.  Parity with the reference is
 * therefore to rounding (tests pin it against golden vectors made by the
 * reference itself), not bitwise.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_CHUNK 256

/* Error codes mirror the reference's checks: 2 <= m <= 16 (_core.pyx:138-139)
 * and the scratch allocation (_core.pyx:141-144). */
int oracle_moment_blocks(const double *xt, int64_t n, int64_t t,
                         const int64_t *col0, const int64_t *edges, int64_t m,
                         double *out, const int64_t *offs, int64_t k0,
                         int64_t k1) {
  (void)n;
  if (m < 2 || m > 16) return 1;
  double *pre = (double *)malloc(sizeof(double) * ORACLE_CHUNK * (size_t)m);
  if (!pre) return 2;
  for (int64_t k = k0; k < k1; ++k) {
    const int64_t *c0 = col0 + k * m;
    const int64_t *e = edges + k * m;
    int64_t nelem = 1;
    for (int64_t q = 0; q < m; ++q) nelem *= e[q];
    int64_t elast = e[m - 1];
    double *blk = out + offs[k];
    /* odometer over the first m-1 modes; the last mode is innermost */
    int64_t o[16];
    for (int64_t s0 = 0; s0 < t; s0 += ORACLE_CHUNK) {
      int64_t cs = t - s0 < ORACLE_CHUNK ? t - s0 : ORACLE_CHUNK;
      memset(o, 0, sizeof(o));
      for (int64_t base = 0; base < nelem; base += elast) {
        /* prefix product over modes 0..m-2 for this chunk */
        const double *x0 = xt + (c0[0] + o[0]) * t + s0;
        for (int64_t s = 0; s < cs; ++s) pre[s] = x0[s];
        for (int64_t q = 1; q < m - 1; ++q) {
          const double *xq = xt + (c0[q] + o[q]) * t + s0;
          for (int64_t s = 0; s < cs; ++s) pre[s] *= xq[s];
        }
        for (int64_t ol = 0; ol < elast; ++ol) {
          const double *xl = xt + (c0[m - 1] + ol) * t + s0;
          double acc = 0.0;
          for (int64_t s = 0; s < cs; ++s) acc += pre[s] * xl[s];
          blk[base + ol] += acc;
        }
        /* advance the odometer over modes m-2 .. 0 */
        for (int64_t q = m - 2; q >= 0; --q) {
          if (++o[q] < e[q]) break;
          o[q] = 0;
        }
      }
    }
  }
  free(pre);
  return 0;
}
