// extern "C" boundary (include/bcgpu.h).  Validation mirrors the reference's
// errors; every launch is stream-ordered on the caller's stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/bcgpu.h"
#include "kernels.h"
#include "plan.h"

struct bcg_plan {
  bcg::Plan p;
};

namespace bcg {
int64_t g_launches = 0;
}

namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char *what) {
  return fail(BCG_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CUDA_TRY(expr, what)                    \
  do {                                          \
    cudaError_t _e = (expr);                    \
    if (_e != cudaSuccess) return cuda_fail(_e, what); \
  } while (0)

// Split-K decision shared by bcg_moment_ws_bytes and bcg_moment_raw: fixed
// kSliceLen-sample slices (association independent of the plan), launched in
// groups whose partials fit the workspace cap.
struct Slicing {
  int KC;
  int nslices;   // total slices
  int group;     // slices per launch
  int64_t slice_len;
};

constexpr int64_t kWsCap = (int64_t)2 << 30;  // 2 GiB of split-K partials at most

Slicing choose_slicing(const bcg::Plan &p, int64_t t) {
  Slicing s{bcg::pick_kc((int)p.n), 1, 1, bcg::kSliceLen};
  if (s.KC == 0 || t <= 0) return s;
  s.nslices = (int)((t + bcg::kSliceLen - 1) / bcg::kSliceLen);
  // slices per launch: as many as the workspace cap allows (fewest launches,
  // no small tail launch), balanced across launches; a plan with enough tiles
  // to fill the GPU by itself (>= 8 waves) runs one slice per launch and
  // accumulates straight into `out` (no workspace, no reduce pass).
  int64_t ntiles = 0;
  for (const bcg::Gemm &g : p.gemm) ntiles += (int64_t)(g.tiles.size() + g.et[0].size() + g.et[1].size());
  ntiles = std::max<int64_t>(1, ntiles);
  const int64_t S = p.S_out;
  int64_t cap = kWsCap / std::max<int64_t>(1, S * 8);
  if (ntiles >= 8 * 148 * 4) cap = 1;
  cap = std::max<int64_t>(1, std::min<int64_t>(cap, s.nslices));
  const int64_t ngroups = (s.nslices + cap - 1) / cap;
  s.group = (int)((s.nslices + ngroups - 1) / ngroups);
  return s;
}

// split-K partials (the transposed-input entries)
size_t ws_bytes_for(const bcg::Plan &p, const Slicing &s) {
  return s.group > 1 ? (size_t)s.group * (size_t)p.S_out * sizeof(double) : 0;
}

// the row-major entries also transpose x into the workspace first
size_t xt_bytes_for(const bcg::Plan &p, int64_t t) {
  return ((size_t)p.n * (size_t)bcg::padded_t(t) * sizeof(double) + 255) / 256 * 256;
}

// xt: transposed data, n rows of stride ldt >= padded_t(t), zero-padded past t
int run_moment(const bcg::Plan &p, const double *xt, int64_t t, int64_t ldt, double *out, void *ws,
               size_t ws_bytes, int64_t k0, int64_t k1, cudaStream_t stream) {
  if (t <= 0) return BCG_OK;
  const Slicing sl = choose_slicing(p, t);
  if (sl.KC == 0) return fail(BCG_EINVAL, "too many columns for the moment kernel's shared-memory stage");
  if (ldt < bcg::padded_t(t) || (ldt & 1) || (reinterpret_cast<uintptr_t>(xt) & 15))
    return fail(BCG_EINVAL, "xt must be 16-byte aligned with an even row stride >= t rounded up to 16");
  const size_t need = ws_bytes_for(p, sl);
  if (need > ws_bytes || (need && !ws))
    return fail(BCG_EINVAL, "workspace too small: need " + std::to_string(need) + " bytes");
  bcg::MomentArgs a{};
  a.x = xt;
  a.t = t;
  a.ldx = ldt;
  a.n = (int)p.n;
  a.offs = p.d_koff;
  a.nslices_total = sl.nslices;
  a.slice_len = sl.slice_len;
  a.out = out;
  a.ws = static_cast<double *>(ws);
  a.S = p.S_out;
  a.kmin_sel = (int32_t)k0;
  a.kmax_sel = k1 - 1 >= INT32_MAX ? INT32_MAX : (int32_t)(k1 - 1);
  if (k0 == 0 && k1 >= p.lay[p.m].K) a.kmax_sel = INT32_MAX;
  const auto &offs = p.lay[p.m].offs;
  const int64_t lo = offs[k0], hi = offs[k1];
  for (int g0 = 0; g0 < sl.nslices; g0 += sl.group) {
    a.slice0 = g0;
    a.nslices = std::min(sl.group, sl.nslices - g0);
    // every GEMM of the plan writes a disjoint set of keys of the same slice
    // partials, so one reduce pass follows them all
    for (const bcg::Gemm &g : p.gemm) {
      if (g.tiles.empty() && g.et[0].empty() && g.et[1].empty()) continue;
      a.h = g.h;
      a.r = g.r;
      a.rowcols = g.d_rowcols;
      a.colcols = g.d_colcols;
      a.row_keybase = g.d_row_keybase;
      a.row_olin = g.d_row_olin;
      a.row_cstart = g.d_row_cstart;
      a.col_rank = g.d_col_rank;
      a.col_olin = g.d_col_olin;
      a.col_size = g.d_col_size;
      a.R = g.R;
      a.C = g.C;
      // the full-width tiles, then the band-edge tiles (tm x ew[0], tm x
      // ew[1]): disjoint elements of the same partials, each summed in the
      // same sample order
      for (int pass = 0; pass < 3; ++pass) {
        const auto &tl = pass == 0 ? g.tiles : g.et[pass - 1];
        if (tl.empty()) continue;
        a.tiles = pass == 0 ? g.d_tiles : g.d_et[pass - 1];
        a.tile_kmin = pass == 0 ? g.d_tile_kmin : g.d_ekmin[pass - 1];
        a.tile_kmax = pass == 0 ? g.d_tile_kmax : g.d_ekmax[pass - 1];
        a.ntiles = (int)tl.size();
        const int64_t grid = (int64_t)a.ntiles * a.nslices;
        if (grid > INT32_MAX) return fail(BCG_EINVAL, "moment grid too large");
        CUDA_TRY(bcg::launch_moment(a, sl.KC, (int)grid, stream, g.tm, pass == 0 ? g.tn : g.ew[pass - 1]),
                 "moment kernel");
        bcg::g_launches++;
      }
    }
    if (a.nslices > 1) {
      CUDA_TRY(bcg::launch_reduce_slices(a.ws, a.nslices, a.S, lo, hi, out, stream),
               "split-K reduce");
      bcg::g_launches++;
    }
  }
  if (p.sym && !p.fill_keys.empty()) {
    // permuted copies inside blocks with repeated block indices
    const auto f0 = std::lower_bound(p.fill_keys.begin(), p.fill_keys.end(), (int32_t)k0) - p.fill_keys.begin();
    const auto f1 = std::lower_bound(p.fill_keys.begin(), p.fill_keys.end(), k1 > INT32_MAX ? INT32_MAX : (int32_t)k1) -
                    p.fill_keys.begin();
    if (f1 > f0) {
      CUDA_TRY(bcg::launch_sym_fill(p.d_fill_keys + f0, f1 - f0, p.d_keys32, p.d_offs, p.m, p.b, p.n, out, stream),
               "symmetric fill");
      bcg::g_launches++;
    }
  }
  return BCG_OK;
}

std::mutex g_cache_mu;
std::map<std::tuple<int64_t, int, int>, std::unique_ptr<bcg_plan>> g_cache;

}  // namespace

extern "C" {

const char *bcg_last_error(void) { return g_err.c_str(); }
int bcg_version(void) { return 100; }
int64_t bcg_launch_count(void) { return bcg::g_launches; }

int bcg_plan_create(int64_t n, int32_t m, int32_t b, bcg_plan **plan) {
  return bcg_plan_create_flags(n, m, b, 0, plan);
}

int bcg_plan_create_ex(int64_t n, int32_t m, int32_t b, int32_t variant, bcg_plan **plan) {
  if (variant > 0) return fail(BCG_EINVAL, "unknown moment kernel variant " + std::to_string(variant));
  return bcg_plan_create_flags(n, m, b, 0, plan);
}

int bcg_plan_create_flags(int64_t n, int32_t m, int32_t b, int32_t flags, bcg_plan **plan) {
  if (!plan) return fail(BCG_EINVAL, "plan pointer is NULL");
  if (flags & ~(BCG_PLAN_FULL | BCG_PLAN_HOST)) return fail(BCG_EINVAL, "unknown plan flags");
  auto pl = std::make_unique<bcg_plan>();
  std::string err = bcg::build_plan(n, m, b, pl->p, -1, !(flags & BCG_PLAN_FULL));
  if (!err.empty()) return fail(BCG_EINVAL, err);
  if (!(flags & BCG_PLAN_HOST)) {
    err = bcg::upload_plan(pl->p);
    if (!err.empty()) {
      bcg::free_plan(pl->p);
      return fail(BCG_ECUDA, err);
    }
  }
  *plan = pl.release();
  return BCG_OK;
}

int bcg_plan_create_host(int64_t n, int32_t m, int32_t b, bcg_plan **plan) {
  return bcg_plan_create_flags(n, m, b, BCG_PLAN_HOST, plan);
}

int bcg_plan_kernel(const bcg_plan *plan, int32_t *variant, int32_t *tm, int32_t *tn, int64_t *ntiles) {
  if (!plan) return fail(BCG_EINVAL, "plan is NULL");
  if (variant) *variant = plan->p.variant;
  // the first (largest) GEMM's tile shape; tiles summed over the GEMMs
  const bcg::Gemm *g0 = plan->p.gemm.empty() ? nullptr : &plan->p.gemm[0];
  if (tm) *tm = g0 ? g0->tm : 0;
  if (tn) *tn = g0 ? g0->tn : 0;
  if (ntiles) {
    *ntiles = 0;
    for (const bcg::Gemm &g : plan->p.gemm) *ntiles += (int64_t)g.tiles.size();
  }
  return BCG_OK;
}

int bcg_plan_gemm(const bcg_plan *plan, int32_t i, int32_t *ngemm, int32_t *split_T, int32_t *info,
                  int64_t *ntiles) {
  if (!plan) return fail(BCG_EINVAL, "plan is NULL");
  const bcg::Plan &p = plan->p;
  if (ngemm) *ngemm = (int32_t)p.gemm.size();
  if (split_T) *split_T = p.split_T;
  if (i < 0) return BCG_OK;
  if (i >= (int32_t)p.gemm.size()) return fail(BCG_EINVAL, "gemm index out of range");
  const bcg::Gemm &g = p.gemm[i];
  if (info) {
    info[0] = g.h;
    info[1] = g.r;
    info[2] = g.tm;
    info[3] = g.tn;
  }
  if (ntiles) *ntiles = (int64_t)g.tiles.size();
  return BCG_OK;
}

int bcg_plan_output(const bcg_plan *plan, int64_t *S_out, int64_t *produced) {
  if (!plan) return fail(BCG_EINVAL, "plan is NULL");
  const bcg::Plan &p = plan->p;
  if (S_out) *S_out = p.S_out;
  if (produced) *produced = p.m < 2 ? 0 : p.produced;
  return BCG_OK;
}

int bcg_plan_tiled(const bcg_plan *plan, int64_t *tiled, int64_t *edge_tiles) {
  if (!plan) return fail(BCG_EINVAL, "plan is NULL");
  int64_t area = 0, ne = 0;
  for (const bcg::Gemm &g : plan->p.gemm) {
    area += (int64_t)g.tiles.size() * g.tm * g.tn;
    for (int i = 0; i < 2; ++i) {
      area += (int64_t)g.et[i].size() * g.tm * g.ew[i];
      ne += (int64_t)g.et[i].size();
    }
  }
  if (tiled) *tiled = area;
  if (edge_tiles) *edge_tiles = ne;
  return BCG_OK;
}

// waste breakdown of the staircase cover (debug / tools/tile_waste.py):
// out[0] = tiled area, out[1] = valid (row, col) pairs inside the tiles (col >=
// the row's first valid column), out[2] = area of the 8 x 8 DMMA sub-tiles
// with no valid pair, out[3] = area of the 32 x 32 warp tiles with no valid
// pair, out[4] = area right of C or below R (overhang)
int bcg_plan_waste(const bcg_plan *plan, int64_t *out) {
  if (!plan || !out) return fail(BCG_EINVAL, "plan / out is NULL");
  for (int i = 0; i < 5; ++i) out[i] = 0;
  for (const bcg::Gemm &g : plan->p.gemm)
    for (int pass = 0; pass < 3; ++pass)
      for (const bcg::Tile &tl : pass == 0 ? g.tiles : g.et[pass - 1]) {
        const int tw = pass == 0 ? g.tn : g.ew[pass - 1];
        out[0] += (int64_t)g.tm * tw;
        auto valid = [&](int64_t r0, int64_t r1, int64_t c0, int64_t c1) {
          int64_t v = 0;
          for (int64_t r = r0; r < std::min<int64_t>(r1, g.R); ++r) {
            const int64_t lo = std::max<int64_t>(c0, g.row_cstart[r]), hi = std::min<int64_t>(c1, g.C);
            if (hi > lo) v += hi - lo;
          }
          return v;
        };
        out[1] += valid(tl.row0, tl.row0 + g.tm, tl.col0, tl.col0 + tw);
        for (int i = 0; i < g.tm; i += 8)
          for (int j = 0; j < tw; j += 8)
            if (!valid(tl.row0 + i, tl.row0 + i + 8, tl.col0 + j, tl.col0 + j + 8)) out[2] += 64;
        for (int i = 0; i < g.tm; i += 32)
          for (int j = 0; j < tw; j += 32)
            if (!valid(tl.row0 + i, tl.row0 + i + 32, tl.col0 + j, tl.col0 + j + std::min(32, tw - j)))
              out[3] += 32 * std::min(32, tw - j);
        for (int64_t r = tl.row0; r < tl.row0 + g.tm; ++r)
          for (int64_t c = tl.col0; c < tl.col0 + tw; ++c)
            if (r >= g.R || c >= g.C) out[4]++;
      }
  return BCG_OK;
}

int bcg_plan_selfcheck(const bcg_plan *plan) {
  if (!plan) return fail(BCG_EINVAL, "plan is NULL");
  const bcg::Plan &p = plan->p;
  if (p.m < 2) return BCG_OK;
  const int64_t S = p.S_out;
  const int o = p.m;
  const bcg::Layout &L = p.lay[o];
  std::vector<uint8_t> seen(S, 0);
  int64_t count = 0;
  for (const bcg::Gemm &g : p.gemm)
  for (int pass = 0; pass < 3; ++pass)
  for (const bcg::Tile &tl : pass == 0 ? g.tiles : g.et[pass - 1]) {
    const int tw = pass == 0 ? g.tn : g.ew[pass - 1];
    for (int64_t r = tl.row0; r < std::min<int64_t>(tl.row0 + g.tm, g.R); ++r) {
      for (int64_t c = tl.col0; c < std::min<int64_t>(tl.col0 + tw, g.C); ++c) {
        if (c < g.row_cstart[r]) continue;
        const int64_t kg = g.row_keybase[r] + g.col_rank[c];
        if (kg < 0 || kg >= (int64_t)p.koff.size()) return fail(BCG_EINVAL, "selfcheck: key index out of range");
        const int64_t lin = (int64_t)g.row_olin[r] * g.col_size[c] + g.col_olin[c];
        const int64_t addr = p.koff[kg] + lin;
        const int64_t k = std::upper_bound(L.offs.begin(), L.offs.end(), addr) - L.offs.begin() - 1;
        if (k < 0 || k >= L.K || addr >= L.offs[k + 1]) return fail(BCG_EINVAL, "selfcheck: offset outside block");
        if (p.koff[kg] != L.offs[k]) return fail(BCG_EINVAL, "selfcheck: element outside its key's block");
        if (seen[addr]) return fail(BCG_EINVAL, "selfcheck: element produced twice");
        seen[addr] = 1;
        ++count;
        int64_t rem = addr - L.offs[k], cols[16];
        for (int q = o - 1; q >= 0; --q) {
          const int64_t e = L.edges[k * o + q];
          cols[q] = L.col0[k * o + q] + rem % e;
          rem /= e;
        }
        // the GEMM element's columns must equal (key, offsets)'s
        int64_t got[16], ng = 0;
        for (int q = 0; q < g.h; ++q) got[ng++] = g.rowcols[r * g.h + q];
        for (int q = 0; q < g.r; ++q) got[ng++] = g.colcols[c * g.r + q];
        if (ng != o) return fail(BCG_EINVAL, "selfcheck: order mismatch");
        for (int q = 0; q < o; ++q)
          if (got[q] != cols[q]) return fail(BCG_EINVAL, "selfcheck: column mismatch");
      }
    }
  }
  if (count != p.produced) return fail(BCG_EINVAL, "selfcheck: produced-element count mismatch");
  // every element must be produced, or (symmetric plan) be a permuted copy of
  // a produced element with digits sorted within runs of equal block indices
  for (int64_t k = 0; k < L.K; ++k) {
    const int64_t *key = &L.keys[k * o];
    const int64_t *e = &L.edges[k * o];
    for (int64_t i = L.offs[k]; i < L.offs[k + 1]; ++i) {
      if (seen[i]) continue;
      if (!p.sym) return fail(BCG_EINVAL, "selfcheck: element never produced");
      int64_t d[16], rem = i - L.offs[k];
      for (int q = o - 1; q >= 0; --q) {
        d[q] = rem % e[q];
        rem /= e[q];
      }
      bool sorted = true;
      for (int q = 1; q < o; ++q) sorted = sorted && !(key[q] == key[q - 1] && d[q] < d[q - 1]);
      if (sorted) return fail(BCG_EINVAL, "selfcheck: sorted element never produced");
      if (!std::binary_search(p.fill_keys.begin(), p.fill_keys.end(), (int32_t)k))
        return fail(BCG_EINVAL, "selfcheck: block with permuted copies missing from the fill list");
    }
  }
  return BCG_OK;
}

int bcg_plan_destroy(bcg_plan *plan) {
  if (!plan) return BCG_OK;
  bcg::free_plan(plan->p);
  delete plan;
  return BCG_OK;
}

int bcg_plan_sizes(const bcg_plan *plan, int32_t order, int64_t *K, int64_t *S) {
  if (!plan || order < 1 || order > plan->p.m) return fail(BCG_EINVAL, "order outside 1..m of the plan");
  const auto &L = plan->p.lay[order];
  if (K) *K = L.K;
  if (S) *S = L.offs.back();
  return BCG_OK;
}

int bcg_plan_layout(const bcg_plan *plan, int32_t order, int64_t *keys, int64_t *col0, int64_t *edges,
                    int64_t *offs) {
  if (!plan || order < 1 || order > plan->p.m) return fail(BCG_EINVAL, "order outside 1..m of the plan");
  const auto &L = plan->p.lay[order];
  if (keys) std::memcpy(keys, L.keys.data(), L.keys.size() * 8);
  if (col0) std::memcpy(col0, L.col0.data(), L.col0.size() * 8);
  if (edges) std::memcpy(edges, L.edges.data(), L.edges.size() * 8);
  if (offs) std::memcpy(offs, L.offs.data(), L.offs.size() * 8);
  return BCG_OK;
}

int bcg_moment_ws_bytes(const bcg_plan *plan, int64_t t, size_t *bytes) {
  if (!plan || !bytes) return fail(BCG_EINVAL, "NULL argument");
  if (plan->p.m < 2) {
    *bytes = 0;
    return BCG_OK;
  }
  *bytes = xt_bytes_for(plan->p, t) + ws_bytes_for(plan->p, choose_slicing(plan->p, t));
  return BCG_OK;
}

int bcg_moment_t_ws_bytes(const bcg_plan *plan, int64_t t, size_t *bytes) {
  if (!plan || !bytes) return fail(BCG_EINVAL, "NULL argument");
  *bytes = plan->p.m < 2 ? 0 : ws_bytes_for(plan->p, choose_slicing(plan->p, t));
  return BCG_OK;
}

size_t bcg_colstats_ws_bytes(int64_t t, int64_t n) {
  if (t < 1 || n < 1) return 0;
  return (2 * (size_t)bcg::colstats_parts(t, n) * n + 1) * sizeof(double);
}

int bcg_colstats(const double *x, int64_t t, int64_t n, int64_t ldx, double *sums, double *mean, double *sumsq,
                 int64_t *first_bad, void *ws, size_t ws_bytes, void *stream) {
  if (t < 1 || n < 1 || ldx < n) return fail(BCG_EINVAL, "data must be non-empty with ldx >= n");
  if (!ws || ws_bytes < bcg_colstats_ws_bytes(t, n))
    return fail(BCG_EINVAL, "workspace too small: need " + std::to_string(bcg_colstats_ws_bytes(t, n)) + " bytes");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int parts = bcg::colstats_parts(t, n);
  cudaError_t e = bcg::launch_colstats(x, t, n, ldx, sums, mean, sumsq, first_bad, static_cast<double *>(ws),
                                       parts, s);
  if (e != cudaSuccess) return cuda_fail(e, "colstats");
  return BCG_OK;
}

int bcg_center(const double *x, int64_t t, int64_t n, int64_t ldx, const double *mean, double *xc, void *stream) {
  if (t < 1 || n < 1 || ldx < n) return fail(BCG_EINVAL, "data must be non-empty with ldx >= n");
  CUDA_TRY(bcg::launch_center(x, t, n, ldx, mean, xc, static_cast<cudaStream_t>(stream)), "center");
  return BCG_OK;
}

// row-major x (t x n, ldx): transpose (zero-padded) into the workspace, then
// the transposed-input GEMM on the rest of the workspace
static int moment_rowmajor(const bcg::Plan &p, const double *x, int64_t t, int64_t ldx, double *out, void *ws,
                           size_t ws_bytes, int64_t k0, int64_t k1, cudaStream_t s) {
  if (t <= 0) return BCG_OK;
  const size_t xtb = xt_bytes_for(p, t);
  if (!ws || ws_bytes < xtb) return fail(BCG_EINVAL, "workspace too small: need at least " + std::to_string(xtb) + " bytes");
  double *xt = static_cast<double *>(ws);
  const int64_t ldt = bcg::padded_t(t);
  CUDA_TRY(bcg::launch_transpose_pad(x, t, p.n, ldx, nullptr, xt, ldt, s), "transpose");
  return run_moment(p, xt, t, ldt, out, static_cast<char *>(ws) + xtb, ws_bytes - xtb, k0, k1, s);
}

int bcg_moment_raw(const bcg_plan *plan, const double *x, int64_t t, int64_t ldx, double *out, void *ws,
                   size_t ws_bytes, void *stream) {
  if (!plan) return fail(BCG_EINVAL, "plan is NULL");
  const bcg::Plan &p = plan->p;
  if (p.m < 2 || p.m > 16) return fail(BCG_EINVAL, "kernel supports 2 <= m <= 16");
  if (ldx < p.n) return fail(BCG_EINVAL, "ldx < n");
  if (!p.d_koff) return fail(BCG_EINVAL, "host-only plan");
  return moment_rowmajor(p, x, t, ldx, out, ws, ws_bytes, 0, p.lay[p.m].K, static_cast<cudaStream_t>(stream));
}

int bcg_moment_raw_t(const bcg_plan *plan, const double *xt, int64_t t, int64_t ldt, double *out, void *ws,
                     size_t ws_bytes, void *stream) {
  if (!plan) return fail(BCG_EINVAL, "plan is NULL");
  const bcg::Plan &p = plan->p;
  if (p.m < 2 || p.m > 16) return fail(BCG_EINVAL, "kernel supports 2 <= m <= 16");
  if (!p.d_koff) return fail(BCG_EINVAL, "host-only plan");
  return run_moment(p, xt, t, ldt, out, ws, ws_bytes, 0, p.lay[p.m].K, static_cast<cudaStream_t>(stream));
}

int bcg_moment_raw_range(const bcg_plan *plan, const double *x, int64_t t, int64_t ldx, double *out, void *ws,
                         size_t ws_bytes, int64_t k0, int64_t k1, void *stream) {
  if (!plan) return fail(BCG_EINVAL, "plan is NULL");
  const bcg::Plan &p = plan->p;
  if (p.m < 2 || p.m > 16) return fail(BCG_EINVAL, "kernel supports 2 <= m <= 16");
  if (ldx < p.n) return fail(BCG_EINVAL, "ldx < n");
  if (!p.d_koff) return fail(BCG_EINVAL, "host-only plan");
  k0 = std::max<int64_t>(k0, 0);
  k1 = std::min<int64_t>(k1, p.lay[p.m].K);
  if (k1 <= k0) return BCG_OK;
  return moment_rowmajor(p, x, t, ldx, out, ws, ws_bytes, k0, k1, static_cast<cudaStream_t>(stream));
}

int bcg_moment_raw_t_range(const bcg_plan *plan, const double *xt, int64_t t, int64_t ldt, double *out, void *ws,
                           size_t ws_bytes, int64_t k0, int64_t k1, void *stream) {
  if (!plan) return fail(BCG_EINVAL, "plan is NULL");
  const bcg::Plan &p = plan->p;
  if (p.m < 2 || p.m > 16) return fail(BCG_EINVAL, "kernel supports 2 <= m <= 16");
  if (!p.d_koff) return fail(BCG_EINVAL, "host-only plan");
  k0 = std::max<int64_t>(k0, 0);
  k1 = std::min<int64_t>(k1, p.lay[p.m].K);
  if (k1 <= k0) return BCG_OK;
  return run_moment(p, xt, t, ldt, out, ws, ws_bytes, k0, k1, static_cast<cudaStream_t>(stream));
}

int bcg_transpose_pad(const double *x, int64_t t, int64_t n, int64_t ldx, const double *mean, double *xt, int64_t ldt,
                      void *stream) {
  if (t < 1 || n < 1 || ldx < n || ldt < t) return fail(BCG_EINVAL, "bad transpose shape");
  CUDA_TRY(bcg::launch_transpose_pad(x, t, n, ldx, mean, xt, ldt, static_cast<cudaStream_t>(stream)), "transpose");
  return BCG_OK;
}

int64_t bcg_padded_t(int64_t t) { return bcg::padded_t(t); }

int bcg_rowstats(const double *xt, int64_t n, int64_t t, int64_t ldt, double *sums, double *sumsq, void *stream) {
  if (t < 1 || n < 1 || ldt < t) return fail(BCG_EINVAL, "bad shape");
  CUDA_TRY(bcg::launch_rowstats(xt, n, t, ldt, sums, sumsq, nullptr, 1, static_cast<cudaStream_t>(stream)),
           "rowstats");
  return BCG_OK;
}

size_t bcg_rowstats_ws_bytes(int64_t n, int64_t t) {
  if (n < 1 || t < 1) return 0;
  return (size_t)n * bcg::rowstats_parts(n, t) * 2 * sizeof(double);
}

int bcg_rowstats_ws(const double *xt, int64_t n, int64_t t, int64_t ldt, double *sums, double *sumsq, void *ws,
                    size_t ws_bytes, void *stream) {
  if (t < 1 || n < 1 || ldt < t) return fail(BCG_EINVAL, "bad shape");
  const int P = bcg::rowstats_parts(n, t);
  if (ws_bytes < (size_t)n * P * 2 * sizeof(double)) return fail(BCG_EINVAL, "rowstats workspace too small");
  CUDA_TRY(bcg::launch_rowstats(xt, n, t, ldt, sums, sumsq, static_cast<double *>(ws), P,
                                static_cast<cudaStream_t>(stream)),
           "rowstats");
  return BCG_OK;
}

int bcg_moment_blocks(const double *xt, int64_t n, int64_t t, const int64_t *col0, const int64_t *edges, int64_t m,
                      int64_t K, double *out, const int64_t *offs, int64_t k0, int64_t k1, void *stream) {
  if (m < 2 || m > 16) return fail(BCG_EINVAL, "kernel supports 2 <= m <= 16");
  if (n < 1 || K < 1) return fail(BCG_EINVAL, "empty layout");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // recover b from the layout: the second key is (1, ..., 1, 2) with col0 = b
  std::vector<int64_t> hc(std::min<int64_t>(K, 2) * m);
  CUDA_TRY(cudaMemcpyAsync(hc.data(), col0, hc.size() * 8, cudaMemcpyDeviceToHost, s), "layout copy");
  CUDA_TRY(cudaStreamSynchronize(s), "layout copy");
  const int64_t b = K >= 2 ? hc[2 * m - 1] : n;
  if (b < 1) return fail(BCG_EINVAL, "layout is not a block layout");
  bcg_plan *pl = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto key = std::make_tuple(n, (int)m, (int)b);
    auto it = g_cache.find(key);
    if (it == g_cache.end()) {
      bcg_plan *np = nullptr;
      // every element computed directly: the reference's per-element
      // accumulate semantics for any prior content of `out`
      int rc = bcg_plan_create_flags(n, (int32_t)m, (int32_t)b, BCG_PLAN_FULL, &np);
      if (rc) return rc;
      it = g_cache.emplace(key, std::unique_ptr<bcg_plan>(np)).first;
    }
    pl = it->second.get();
  }
  const bcg::Layout &L = pl->p.lay[m];
  if (L.K != K) return fail(BCG_EINVAL, "layout does not match _block_layout(n, m, b)");
  {
    std::vector<int64_t> hc0(K * m), he(K * m), ho(K + 1);
    CUDA_TRY(cudaMemcpyAsync(hc0.data(), col0, hc0.size() * 8, cudaMemcpyDeviceToHost, s), "layout copy");
    CUDA_TRY(cudaMemcpyAsync(he.data(), edges, he.size() * 8, cudaMemcpyDeviceToHost, s), "layout copy");
    CUDA_TRY(cudaMemcpyAsync(ho.data(), offs, ho.size() * 8, cudaMemcpyDeviceToHost, s), "layout copy");
    CUDA_TRY(cudaStreamSynchronize(s), "layout copy");
    if (hc0 != L.col0 || he != L.edges || ho != L.offs)
      return fail(BCG_EINVAL, "layout does not match _block_layout(n, m, b)");
  }
  k0 = std::max<int64_t>(k0, 0);
  k1 = std::min<int64_t>(k1, K);
  if (k1 <= k0 || t <= 0) return BCG_OK;
  // the reference's signature has no workspace: stream-ordered allocations
  // from the device pool, kept mapped between calls (no trim at each sync)
  {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  double *x = nullptr;
  void *ws = nullptr;
  const size_t wsb = ws_bytes_for(pl->p, choose_slicing(pl->p, t));
  const int64_t ldt = bcg::padded_t(t);
  CUDA_TRY(cudaMallocAsync(&x, (size_t)ldt * n * sizeof(double), s), "padded copy");
  if (wsb) {
    cudaError_t e = cudaMallocAsync(&ws, wsb, s);
    if (e != cudaSuccess) {
      cudaFreeAsync(x, s);
      return cuda_fail(e, "workspace");
    }
  }
  // the reference's xt is already the transposed layout; pad its rows to ldt
  cudaError_t e = bcg::launch_pad_rows(xt, n, t, t, x, ldt, s);
  int rc = e == cudaSuccess ? run_moment(pl->p, x, t, ldt, out, ws, wsb, k0, k1, s) : cuda_fail(e, "pad copy");
  cudaFreeAsync(x, s);
  if (ws) cudaFreeAsync(ws, s);
  return rc;
}

static int recursion_common(const bcg_plan *plan, double *mk, const double *const *lower, int mode, int sigma_lo,
                            int sigma_hi, int64_t k0, int64_t k1, cudaStream_t s, const int32_t *klist = nullptr,
                            int64_t e0 = 0, int64_t e1 = INT64_MAX) {
  const bcg::Plan &p = plan->p;
  if (!p.d_offs) return fail(BCG_EINVAL, "host-only plan");
  bcg::RecursionArgs a{};
  a.m = p.m;
  a.b = p.b;
  a.n = p.n;
  a.K = p.lay[p.m].K;
  a.offs = p.d_offs;
  a.keys = p.d_keys32;
  a.sub_rank = p.d_sub_rank;
  a.part_mask = p.d_part_mask;
  a.nslots = p.nslots;
  for (int sg = 0; sg < (int)p.sigma_first.size() && sg < 12; ++sg) a.sigma_first[sg] = p.sigma_first[sg];
  a.sigma_lo = sigma_lo;
  a.sigma_hi = sigma_hi;
  a.p_begin = p.sigma_first[sigma_lo];
  a.p_end = p.sigma_first[sigma_hi + 1];
  // orders the processed partitions actually read (bc/cumulants.py:65-66)
  bool needed[17] = {false};
  for (int q = a.p_begin; q < a.p_end; ++q)
    for (int i = 0; i < 8; ++i)
      if (p.part_mask[q * 8 + i]) needed[__builtin_popcount(p.part_mask[q * 8 + i])] = true;
  for (int k = 2; k <= p.m - 2; ++k) {
    a.lower_offs[k] = p.d_lower_offs[k];
    a.lower[k] = lower ? lower[k - 2] : nullptr;
    if (needed[k] && !a.lower[k])
      return fail(BCG_EINVAL, "missing lower cumulant of order " + std::to_string(k));
  }
  a.mk = mk;
  a.mode = mode;
  a.e0 = e0;
  a.e1 = e1;
  a.k0 = std::max<int64_t>(0, k0);
  a.k1 = std::min<int64_t>(a.K, k1);
  a.klist = klist;
  CUDA_TRY(bcg::launch_recursion(a, s), "recursion kernel");
  return BCG_OK;
}

// Recursion dispatcher: the factored register-blocked kernel (recursion_fact.cu)
// for full blocks when the plan supports it and the central moments it needs
// are given; the partition-table kernel (recursion.cu) for everything else.
static int recursion_dispatch(const bcg_plan *plan, double *mk, const double *const *lower,
                              const double *const *cmom, int64_t k0, int64_t k1, cudaStream_t s) {
  const bcg::Plan &p = plan->p;
  if (p.m <= 3) return BCG_OK;
  if (!p.d_offs) return fail(BCG_EINVAL, "host-only plan");
  const int m = p.m;
  k0 = std::max<int64_t>(0, k0);
  k1 = std::min<int64_t>(p.lay[m].K, k1);
  if (k1 <= k0) return BCG_OK;
  static const bool force_partition = getenv("BCG_RECURSION_PARTITION") != nullptr;  // A/B knob
  bool fact = p.fact_terms > 0 && lower && !force_partition;
  for (int k = 4; fact && k <= m - 2; ++k) fact = cmom && cmom[k - 2];
  if (!fact) return recursion_common(plan, mk, lower, 0, 2, m / 2, k0, k1, s);
  for (int k = 2; k <= m - 2; ++k)
    if (!lower[k - 2]) return fail(BCG_EINVAL, "missing lower cumulant of order " + std::to_string(k));
  bcg::RecFactArgs a{};
  a.term_off = p.d_term_off;
  for (int k = 2; k <= m - 2; ++k) {
    a.cum[k] = lower[k - 2];
    if (k >= 4) a.cmom[k] = cmom[k - 2];
  }
  a.mk = mk;
  auto lo_f = std::lower_bound(p.full_keys.begin(), p.full_keys.end(), (int32_t)k0) - p.full_keys.begin();
  auto hi_f = std::lower_bound(p.full_keys.begin(), p.full_keys.end(), (int32_t)k1) - p.full_keys.begin();
  a.blk_off = p.d_full_offs + lo_f;
  a.term_off = p.d_term_off + lo_f * 2 * p.fact_terms;
  a.nkeys = hi_f - lo_f;
  // whole work list: the tail-grouped order (v7 reloads its second factors
  // only when the key's modes 1..5 change); a sub-range keeps the list order
  if (lo_f == 0 && hi_f == (int64_t)p.full_keys.size()) {
    a.order = p.d_tail_order;
    a.newv = p.d_tail_new;
  }
  if (a.nkeys > 0) CUDA_TRY(bcg::launch_recursion_fact(a, m, p.b, s), "factored recursion kernel");
  auto lo_p = std::lower_bound(p.partial_keys.begin(), p.partial_keys.end(), (int32_t)k0) - p.partial_keys.begin();
  auto hi_p = std::lower_bound(p.partial_keys.begin(), p.partial_keys.end(), (int32_t)k1) - p.partial_keys.begin();
  if (hi_p > lo_p) {
    // partial-edge blocks: partition kernel over the explicit key list
    return recursion_common(plan, mk, lower, 0, 2, m / 2, 0, hi_p - lo_p, s, p.d_partial_keys + lo_p);
  }
  return BCG_OK;
}

int bcg_cumulant_recursion(const bcg_plan *plan, double *mk, const double *const *lower, void *stream) {
  if (!plan) return fail(BCG_EINVAL, "plan is NULL");
  return recursion_dispatch(plan, mk, lower, nullptr, 0, plan->p.lay[plan->p.m].K, static_cast<cudaStream_t>(stream));
}

int bcg_cumulant_recursion_range(const bcg_plan *plan, double *mk, const double *const *lower, int64_t k0,
                                 int64_t k1, void *stream) {
  if (!plan) return fail(BCG_EINVAL, "plan is NULL");
  return recursion_dispatch(plan, mk, lower, nullptr, k0, k1, static_cast<cudaStream_t>(stream));
}

int bcg_cumulant_recursion_ex(const bcg_plan *plan, double *mk, const double *const *lower,
                              const double *const *cmom, int64_t k0, int64_t k1, void *stream) {
  if (!plan) return fail(BCG_EINVAL, "plan is NULL");
  return recursion_dispatch(plan, mk, lower, cmom, k0, k1, static_cast<cudaStream_t>(stream));
}

int bcg_cumulant_recursion_span(const bcg_plan *plan, double *mk, const double *const *lower,
                                const double *const *cmom, int64_t e0, int64_t e1, void *stream) {
  if (!plan) return fail(BCG_EINVAL, "plan is NULL");
  const bcg::Plan &p = plan->p;
  if (p.m <= 3) return BCG_OK;
  const auto &offs = p.lay[p.m].offs;
  const int64_t K = p.lay[p.m].K;
  e0 = std::max<int64_t>(e0, 0);
  e1 = std::min<int64_t>(e1, offs[K]);
  if (e1 <= e0) return BCG_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // blocks entirely inside the span: the regular dispatch (factored kernel)
  const int64_t ka = std::lower_bound(offs.begin(), offs.end(), e0) - offs.begin();         // offs[ka] >= e0
  const int64_t kb = std::upper_bound(offs.begin(), offs.end(), e1) - offs.begin() - 1;     // offs[kb] <= e1
  if (kb > ka) {
    const int rc = recursion_dispatch(plan, mk, lower, cmom, ka, kb, s);
    if (rc) return rc;
  }
  // the (at most two) blocks cut by the span's ends: partition kernel with
  // writes masked to [e0, e1)
  int64_t cut[2] = {-1, -1};
  if (offs[ka] > e0) cut[0] = ka - 1;                          // block holding e0
  if (kb < K && offs[kb] < e1 && kb != cut[0]) cut[1] = kb;    // block holding e1 - 1
  for (int64_t k : cut) {
    if (k < 0) continue;
    const int rc = recursion_common(plan, mk, lower, 0, 2, p.m / 2, k, k + 1, s, nullptr, e0, e1);
    if (rc) return rc;
  }
  return BCG_OK;
}

int bcg_outer_prod_cum(const bcg_plan *plan, int32_t sigma, const double *const *lower, double *out, void *stream) {
  if (!plan) return fail(BCG_EINVAL, "plan is NULL");
  if (sigma < 2 || sigma > plan->p.m / 2)
    return fail(BCG_EINVAL, "sigma must be in 2..m//2=" + std::to_string(plan->p.m / 2) + ", got " +
                                std::to_string(sigma));
  return recursion_common(plan, out, lower, 1, sigma, sigma, 0, plan->p.lay[plan->p.m].K,
                          static_cast<cudaStream_t>(stream));
}

int bcg_axpby(int64_t len, double a, const double *x, double c, const double *y, double *out, void *stream) {
  CUDA_TRY(bcg::launch_axpby(len, a, x, c, y, out, static_cast<cudaStream_t>(stream)), "axpby");
  return BCG_OK;
}

int bcg_div(int64_t len, const double *x, double d, double *out, void *stream) {
  CUDA_TRY(bcg::launch_div(len, x, d, out, static_cast<cudaStream_t>(stream)), "div");
  return BCG_OK;
}

size_t bcg_dense_subsets_ws_bytes(int64_t E, int32_t m, int64_t t) {
  if (E <= 0 || m < 1 || m > 8) return 0;
  return (size_t)E * (size_t)bcg::dense_subsets_parts(E, t) * ((size_t)1 << m) * sizeof(double);
}

int bcg_dense_subsets(const double *x, int64_t t, int64_t n, int64_t ldx, const double *mean, int32_t m,
                      const int32_t *idx, int64_t E, double *out, void *ws, size_t ws_bytes, void *stream) {
  if (m < 1 || m > 8) return fail(BCG_EINVAL, "dense entries support 1 <= m <= 8");
  if (t <= 0 || n <= 0 || ldx < n) return fail(BCG_EINVAL, "bad data shape");
  if (E <= 0) return BCG_OK;
  if (!x || !mean || !idx || !out) return fail(BCG_EINVAL, "NULL pointer");
  const size_t need = bcg_dense_subsets_ws_bytes(E, m, t);
  if (!ws || ws_bytes < need) return fail(BCG_EINVAL, "workspace too small: need " + std::to_string(need) + " bytes");
  CUDA_TRY(bcg::launch_dense_subsets(x, t, n, ldx, mean, m, idx, E, static_cast<double *>(ws),
                                     bcg::dense_subsets_parts(E, t), out, static_cast<cudaStream_t>(stream)),
           "dense subsets");
  return BCG_OK;
}

}  // extern "C"
