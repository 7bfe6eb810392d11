// Host-side plan construction: the reference layout (bc/_engines.py:46-54),
// the Khatri-Rao GEMM tables of the order-m moment, the staircase tile list
// and the recursion's partition / sub-block tables.  Runs once per (n, m, b).
#include "plan.h"

#include <cuda_runtime.h>

#include "kernels.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <numeric>

namespace bcg {

static int64_t binom(int64_t a, int64_t c) {
  if (c < 0 || a < c) return 0;
  int64_t r = 1;
  for (int64_t i = 0; i < c; ++i) r = r * (a - i) / (i + 1);
  return r;
}

// Rank of a sorted 1-based k-tuple among all sorted k-tuples over 1..nbar in
// lexicographic (combinations_with_replacement) order, bc/symtensor.py:47-49:
//   sum_q sum_{v = j_{q-1}}^{j_q - 1} C(nbar - v + k - q, k - q),  j_0 = 1.
int64_t multiset_rank(const int64_t *key, int k, int64_t nbar) {
  int64_t rank = 0, prev = 1;
  for (int q = 1; q <= k; ++q) {
    for (int64_t v = prev; v < key[q - 1]; ++v) rank += binom(nbar - v + k - q, k - q);
    prev = key[q - 1];
  }
  return rank;
}

static void enum_sorted(int64_t nbar, int k, std::vector<int64_t> &out) {
  // lexicographic sorted k-tuples: odometer that resets the tail to the
  // incremented digit (combinations_with_replacement order)
  std::vector<int64_t> key(k, 1);
  if (k == 0) return;
  while (true) {
    out.insert(out.end(), key.begin(), key.end());
    int q = k - 1;
    while (q >= 0 && key[q] == nbar) --q;
    if (q < 0) break;
    ++key[q];
    for (int i = q + 1; i < k; ++i) key[i] = key[q];
  }
}

static inline int64_t edge_of(int64_t j, int64_t n, int64_t b) {
  return std::min(j * b, n) - (j - 1) * b;
}

static void build_layout(int64_t n, int b, int64_t nbar, int order, Layout &L) {
  L.order = order;
  L.keys.clear();
  enum_sorted(nbar, order, L.keys);
  L.K = (int64_t)L.keys.size() / order;
  L.col0.resize(L.keys.size());
  L.edges.resize(L.keys.size());
  L.offs.assign(L.K + 1, 0);
  for (int64_t k = 0; k < L.K; ++k) {
    int64_t size = 1;
    for (int q = 0; q < order; ++q) {
      int64_t j = L.keys[k * order + q];
      L.col0[k * order + q] = (j - 1) * b;
      L.edges[k * order + q] = edge_of(j, n, b);
      size *= L.edges[k * order + q];
    }
    L.offs[k + 1] = L.offs[k] + size;
  }
}

// Canonical min-2 partitions of (1..m) into sigma parts, the reference's
// enumeration order (bc/partitions.py:63-98): element e joins each open part
// in opening order, then opens a new one; prune when the remaining elements
// cannot complete every short / unopened part.
std::vector<std::vector<std::vector<int>>> partitions_min2(int m, int sigma) {
  std::vector<std::vector<std::vector<int>>> out;
  std::vector<std::vector<int>> parts;
  std::function<void(int, int)> rec = [&](int e, int shortc) {
    int left = m - e + 1;
    if (e > m) {
      if ((int)parts.size() == sigma && shortc == 0) out.push_back(parts);
      return;
    }
    if (left < shortc + 2 * (sigma - (int)parts.size())) return;
    for (size_t i = 0; i < parts.size(); ++i) {
      bool single = parts[i].size() == 1;
      parts[i].push_back(e);
      rec(e + 1, shortc - (single ? 1 : 0));
      parts[i].pop_back();
    }
    if ((int)parts.size() < sigma) {
      parts.push_back({e});
      rec(e + 1, shortc + 1);
      parts.pop_back();
    }
  };
  rec(1, 0);
  return out;
}

static void build_fact_tables(Plan &p);

int default_variant() {  // only the v1 kernel family (variant 0) remains
  const char *env = std::getenv("BCG_MOMENT_VARIANT");
  if (env && *env) return std::atoi(env);
  return 0;
}

// Staircase tile lists of GEMM g for a tm x tn CTA tile.  Every band of tm
// rows is covered from its first row's suffix start by tiles of width
// w[0] = tn; its tail by the narrower widths w[1] = tn/2, w[2] = tn/4 where
// those are compiled shapes (0 = not available): a tail of R < tn columns
// takes one tn tile if R > w[1] + w[2], else w[1] (then w[2]) or w[2] alone
// -- at most w[2] - 1 (or w[1] - 1) masked columns instead of up to tn - 1.
// out (3 classes, or null) receives each class's tiles and key ranges;
// returns the modeled cost: sum over tiles of tm x w x (1 + 10 (1/w + 1/tm))
// (a Khatri-Rao product ~ 10 FMA-equivalents: its X loads, DMULs on the
// shared FP64 pipe, the smem store; fitted to profiles/r01_tile_shapes.log).
struct TileLists {
  std::vector<Tile> t;
  std::vector<int32_t> kmin, kmax;
};
static double build_tiles(const Plan &p, const Gemm &g, int tm, const int (&w)[3], TileLists *out) {
  (void)p;
  if (out)
    for (int i = 0; i < 3; ++i) out[i] = TileLists();
  double cost = 0.0;
  for (int64_t r0 = 0; r0 < g.R; r0 += tm) {
    const int64_t r1 = std::min<int64_t>(r0 + tm, g.R);
    int64_t c0 = g.row_cstart[r0];
    while (c0 < g.C) {
      const int64_t rem = g.C - c0;
      int cls = 0;
      if (rem < w[0]) {
        if (w[1] && rem <= w[1]) cls = (w[2] && rem <= w[2]) ? 2 : 1;
        else if (w[1] && w[2] && rem <= w[1] + w[2]) cls = 1;
      }
      const int tw = w[cls];
      const int64_t c1 = std::min<int64_t>(c0 + tw, g.C);
      cost += (double)tm * tw * (1.0 + 10.0 * (1.0 / tw + 1.0 / tm));
      if (out) {
        // key range of the tile (column ranks are not monotone in a
        // symmetric plan's column order); rows of equal start share it
        int64_t kmin = INT64_MAX, kmax = -1;
        int32_t rlo = 0, rhi = -1;
        for (int64_t rr = r0; rr < r1; ++rr) {
          const int64_t cs = std::max<int64_t>(c0, g.row_cstart[rr]);
          if (cs >= c1) continue;
          if (rr == r0 || g.row_cstart[rr] != g.row_cstart[rr - 1]) {
            rlo = INT32_MAX;
            rhi = -1;
            for (int64_t c = cs; c < c1; ++c) {
              rlo = std::min(rlo, g.col_rank[c]);
              rhi = std::max(rhi, g.col_rank[c]);
            }
          }
          kmin = std::min<int64_t>(kmin, g.row_keybase[rr] + rlo);
          kmax = std::max<int64_t>(kmax, g.row_keybase[rr] + rhi);
        }
        if (kmax >= 0) {
          out[cls].t.push_back(Tile{(int32_t)r0, (int32_t)c0});
          out[cls].kmin.push_back((int32_t)kmin);
          out[cls].kmax.push_back((int32_t)kmax);
        }
      }
      c0 += tw;
    }
  }
  return cost;
}

// tile widths of a tm x tn plan: tn and the compiled narrower edge shapes
static void tile_widths(const Plan &p, int m, int tm, int tn, int (&w)[3]) {
  const int kc = pick_kc((int)p.n);
  w[0] = tn;
  w[1] = (!std::getenv("BCG_NO_EDGE_TILES") && tn / 2 >= 8 && v1_shape_supported(kc, m, tm, tn / 2)) ? tn / 2 : 0;
  w[2] = (w[1] && tn / 4 >= 8 && v1_shape_supported(kc, m, tm, tn / 4)) ? tn / 4 : 0;
}

static double gemm_cost(const Plan &p, const Gemm &g, int tm, int tn) {
  int w[3];
  tile_widths(p, g.h + g.r, tm, tn, w);
  return build_tiles(p, g, tm, w, nullptr);
}

static void choose_shape(const Plan &p, Gemm &g) {
  g.tm = kTM;
  g.tn = kTN;
  const int m = g.h + g.r;
  const char *env = std::getenv("BCG_TILE");
  int etm = 0, etn = 0;
  if (env && std::sscanf(env, "%dx%d", &etm, &etn) == 2 && v1_shape_supported(pick_kc((int)p.n), m, etm, etn)) {
    g.tm = etm;
    g.tn = etn;
    return;
  }
  if (pick_kc((int)p.n) != 16 || m < 2 || m > 8) return;
  // 64 x 128 before 128 x 64 (equal modeled cost; measured 1% faster at the
  // cfg5 order-6 staircase, profiles/r02_moment_experiments.log (8))
  static const int shapes[][2] = {{64, 64}, {16, 128}, {128, 16}, {32, 64}, {64, 32}, {32, 32}, {64, 128}, {128, 64}};
  double best = gemm_cost(p, g, 64, 64);
  // 8-warp shapes (64 x 128, 128 x 64) halve one dimension's Khatri-Rao build
  // per FMA: a win where the build is expensive (three-mode factors on both
  // sides: cfg5 order 6 -7.3%), a loss for two-mode factors (cfg3 order 5's
  // (2|3) GEMM: +2%); BCG_NO_WIDE_TILES=1 disables them (A/B knob)
  static const bool no_wide = std::getenv("BCG_NO_WIDE_TILES") != nullptr;
  const bool wide_ok = !no_wide && g.h >= 3 && g.r >= 3;
  for (const auto &sh : shapes) {
    if (!wide_ok && sh[0] * sh[1] >= 8192) continue;
    const double c = gemm_cost(p, g, sh[0], sh[1]);
    if (c < best * 0.97) {  // switch only for a clear modeled gain
      best = c;
      g.tm = sh[0];
      g.tn = sh[1];
    }
  }
}

// In-block offsets of a sorted block tuple T (len k) that a GEMM row / column
// produces, row-major over its edges: all of them, or (sym) those whose digits
// are non-decreasing within every run of equal block indices -- the other
// offsets of such a run are permutations of one of these (the tensor is
// super-symmetric) and are filled from it after the GEMM (k_sym_fill).
static void tuple_offsets(const int64_t *T, int k, const std::vector<int64_t> &sym_edge, bool sym,
                          std::vector<int64_t> &out) {
  out.clear();
  int64_t e[16], sz = 1;
  for (int q = 0; q < k; ++q) sz *= (e[q] = sym_edge[T[q]]);
  int64_t d[16] = {0};
  for (int64_t o = 0; o < sz; ++o) {
    bool canon = true;
    if (sym)
      for (int q = 1; q < k && canon; ++q) canon = !(T[q] == T[q - 1] && d[q] < d[q - 1]);
    if (canon) out.push_back(o);
    for (int q = k - 1; q >= 0; --q) {  // row-major odometer
      if (++d[q] < e[q]) break;
      d[q] = 0;
    }
  }
}

// GEMM tables over the block alphabet 1..N (sym_edge / sym_col0): rows =
// sorted h-tuples L with one row per produced in-block offset, cols = sorted
// (m-h)-tuples R likewise; (L, R) is a stored key when R[0] >= v = L[h-1].
// Each tuple contributes one row / column per produced in-block offset
// (tuple_offsets); row_olin / col_olin keep the full row-major offset, so the
// epilogue address of an element is the same for every plan.
//
// Full plan: rows grouped by v, columns lexicographic -- row group v is valid
// from the first column whose tuple starts with >= max(v, tcol).
//
// Symmetric plan: a run of equal block indices may straddle the L | R split
// (L ends with v, R starts with v); the element is canonical (digits
// non-decreasing within every run of the full key) iff additionally the last
// digit of L <= the first digit of R.  Columns are ordered by (R[0], first
// digit) and rows by their valid-column start, so row (v, d) is valid on the
// suffix {R[0] > v} + {R[0] == v, first digit >= d}: the GEMM produces exactly
// the canonical elements (C(n+m-1, m) of them when b | n) and k_sym_fill
// copies every other stored element from its canonical permutation.
static std::string build_gemm(Plan &p, Gemm &g, const std::vector<int64_t> &sym_edge,
                              const std::vector<int64_t> &sym_col0, int64_t N, int h, int64_t vmax,
                              int64_t tcol) {
  const int m = p.m;
  g.h = h;
  g.r = m - h;
  const int r = g.r;
  std::vector<int64_t> lt, rt, offs;
  enum_sorted(N, h, lt);
  enum_sorted(N, r, rt);
  const int64_t NL = (int64_t)lt.size() / h, NR = (int64_t)rt.size() / r;
  // ---- columns: (tuple, offset) pairs ----
  struct Col {
    int64_t tuple, off, first_digit;
  };
  std::vector<Col> cols;
  for (int64_t i = 0; i < NR; ++i) {
    const int64_t *Rt = &rt[i * r];
    int64_t tail = 1;  // size of the modes after the first
    for (int q = 1; q < r; ++q) tail *= sym_edge[Rt[q]];
    tuple_offsets(Rt, r, sym_edge, p.sym, offs);
    for (int64_t o : offs) cols.push_back(Col{i, o, o / tail});
  }
  if (p.sym)  // (R[0], first digit), then lexicographic (tuple, offset)
    std::stable_sort(cols.begin(), cols.end(), [&](const Col &a, const Col &c) {
      const int64_t fa = rt[a.tuple * r], fc = rt[c.tuple * r];
      return fa != fc ? fa < fc : a.first_digit < c.first_digit;
    });
  g.C = (int64_t)cols.size();
  g.colcols.resize(g.C * r);
  g.col_rank.resize(g.C);
  g.col_olin.resize(g.C);
  g.col_size.resize(g.C);
  for (int64_t c = 0; c < g.C; ++c) {
    const int64_t *Rt = &rt[cols[c].tuple * r];
    int64_t e[16], sz = 1;
    for (int q = 0; q < r; ++q) sz *= (e[q] = sym_edge[Rt[q]]);
    int64_t rem = cols[c].off;
    for (int q = r - 1; q >= 0; --q) {
      g.colcols[c * r + q] = (int16_t)(sym_col0[Rt[q]] + rem % e[q]);
      rem /= e[q];
    }
    g.col_rank[c] = (int32_t)cols[c].tuple;
    g.col_olin[c] = (int32_t)cols[c].off;
    g.col_size[c] = (int32_t)sz;
  }
  // first column of the suffix valid for a row ending in block v with last
  // digit d (d = -1: no digit condition, i.e. R[0] >= v)
  auto cstart = [&](int64_t v, int64_t d) -> int64_t {
    int64_t lo = 0, hi = g.C;  // first c with (R[0], first digit) >= (v, max(d, 0))
    const int64_t dd = d < 0 ? 0 : d;
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      const int64_t f = rt[cols[mid].tuple * r];
      const bool before = p.sym ? (f < v || (f == v && cols[mid].first_digit < dd)) : f < v;
      if (before) lo = mid + 1;
      else hi = mid;
    }
    return lo;
  };
  std::vector<int64_t> rank_first_v(N + 2, NR);
  for (int64_t v = 1; v <= N; ++v) {
    std::vector<int64_t> vv(r, v);
    rank_first_v[v] = multiset_rank(vv.data(), r, N);
  }
  // full plan: columns lexicographic, so the suffix search above (on R[0]
  // only) is exact; symmetric plan: rows sorted by their suffix start
  struct Row {
    int64_t tuple, off, cs;
  };
  std::vector<Row> rows;
  for (int64_t i = 0; i < NL; ++i) {
    const int64_t *L = &lt[i * h];
    const int64_t v = L[h - 1];
    if (v > vmax) continue;
    const int64_t vc = std::max(v, tcol);
    tuple_offsets(L, h, sym_edge, p.sym, offs);
    for (int64_t o : offs) {
      // the digit condition applies only when R may start with v itself
      const int64_t cs = (p.sym && vc == v) ? cstart(v, o % sym_edge[v]) : cstart(vc, -1);
      if (cs >= g.C) continue;
      rows.push_back(Row{i, o, cs});
    }
  }
  // (suffix start, last entry, lexicographic): non-decreasing starts, so a
  // tile's first row has the earliest valid column of its row band
  std::stable_sort(rows.begin(), rows.end(), [&](const Row &a, const Row &c) {
    if (a.cs != c.cs) return a.cs < c.cs;
    return lt[a.tuple * h + h - 1] < lt[c.tuple * h + h - 1];
  });
  g.R = (int64_t)rows.size();
  g.rowcols.resize(g.R * h);
  g.row_keybase.resize(g.R);
  g.row_olin.resize(g.R);
  g.row_cstart.resize(g.R);
  for (int64_t row = 0; row < g.R; ++row) {
    const int64_t *L = &lt[rows[row].tuple * h];
    const int64_t v = L[h - 1];
    int64_t full[16], e[16];
    for (int q = 0; q < h; ++q) full[q] = L[q];
    for (int q = h; q < m; ++q) full[q] = v;
    const int64_t kbase = multiset_rank(full, m, N) - rank_first_v[v];
    for (int q = 0; q < h; ++q) e[q] = sym_edge[L[q]];
    int64_t rem = rows[row].off;
    for (int q = h - 1; q >= 0; --q) {
      g.rowcols[row * h + q] = (int16_t)(sym_col0[L[q]] + rem % e[q]);
      rem /= e[q];
    }
    g.row_keybase[row] = (int32_t)kbase;
    g.row_olin[row] = (int32_t)rows[row].off;
    g.row_cstart[row] = (int32_t)rows[row].cs;
  }
  if (g.R > INT32_MAX || g.C > INT32_MAX) return "GEMM dimension overflow";
  return "";
}

static int64_t gemm_produced(const Gemm &g) {
  int64_t s = 0;
  for (int64_t r = 0; r < g.R; ++r) s += g.C - g.row_cstart[r];
  return s;
}

std::string build_plan(int64_t n, int m, int b, Plan &p, int variant, bool sym) {
  if (n < 1 || m < 1 || b < 1) return "n, m and b must all be >= 1";
  p.sym = sym;
  p.variant = variant < 0 ? default_variant() : variant;
  if (m > 16) return "kernel supports 2 <= m <= 16";
  p.n = n;
  p.m = m;
  p.b = b;
  p.nbar = (n + b - 1) / b;
  if (n > 32767) return "n > 32767 columns is not supported";
  p.lay.assign(m + 1, Layout());
  for (int k = 1; k <= m; ++k) build_layout(n, b, p.nbar, k, p.lay[k]);
  const Layout &LM = p.lay[m];
  if (LM.offs.back() > (int64_t)INT32_MAX * 64) return "tensor too large";
  if (LM.K > INT32_MAX) return "too many blocks";
  if (m < 2) return "";
  for (int64_t k = 0; k < LM.K; ++k)
    if (LM.offs[k + 1] - LM.offs[k] > INT32_MAX) return "block too large";

  // ---- moment GEMM tables over the block alphabet 1..nbar ----
  const int64_t N = p.nbar;
  std::vector<int64_t> sym_edge(N + 1, 0), sym_col0(N + 1, 0);  // 1-based
  for (int64_t j = 1; j <= N; ++j) {
    sym_edge[j] = edge_of(j, n, b);
    sym_col0[j] = (j - 1) * b;
  }
  p.koff.assign(LM.offs.begin(), LM.offs.end() - 1);  // GEMM key k = layout key k
  p.S_out = LM.offs.back();
  // ---- the GEMM(s) ----
  // odd m: try the hybrid split of the keys by their middle entry
  // (key[h] < T: (h+1 | r-1) GEMM; else (h | r)), pick the T whose 64 x 64
  // tiling covers the staircase with the least area (independent of the tile
  // shapes chosen below, so every shape gives the same factorization)
  const int h0 = m / 2;
  p.gemm.assign(1, Gemm());
  p.split_T = 0;
  {
    std::string err = build_gemm(p, p.gemm[0], sym_edge, sym_col0, N, h0, N, 1);
    if (!err.empty()) return err;
  }
  if ((m % 2) == 1 && m >= 3 && !std::getenv("BCG_NO_HYBRID")) {
    double best = gemm_cost(p, p.gemm[0], 64, 64);
    for (int64_t T = 2; T <= N; ++T) {
      Gemm ga, gb;
      if (!build_gemm(p, ga, sym_edge, sym_col0, N, h0, N, T).empty()) continue;
      if (!build_gemm(p, gb, sym_edge, sym_col0, N, h0 + 1, T - 1, 1).empty()) continue;
      const double c = (ga.R ? gemm_cost(p, ga, 64, 64) : 0.0) + (gb.R ? gemm_cost(p, gb, 64, 64) : 0.0);
      if (c < best * 0.97) {
        best = c;
        p.split_T = (int)T;
      }
    }
    if (p.split_T) {
      p.gemm.assign(2, Gemm());
      build_gemm(p, p.gemm[0], sym_edge, sym_col0, N, h0, N, p.split_T);
      build_gemm(p, p.gemm[1], sym_edge, sym_col0, N, h0 + 1, p.split_T - 1, 1);
      if (p.gemm[1].R == 0) p.gemm.pop_back();
      if (p.gemm[0].R == 0) p.gemm.erase(p.gemm.begin());
    }
  }
  // per-GEMM CTA tile shape (tile model) and tile lists
  p.produced = 0;
  for (Gemm &g : p.gemm) {
    choose_shape(p, g);
    int w[3];
    tile_widths(p, m, g.tm, g.tn, w);
    TileLists tl[3];
    build_tiles(p, g, g.tm, w, tl);
    g.tiles = std::move(tl[0].t);
    g.tile_kmin = std::move(tl[0].kmin);
    g.tile_kmax = std::move(tl[0].kmax);
    for (int i = 0; i < 2; ++i) {
      g.ew[i] = w[i + 1];
      g.et[i] = std::move(tl[i + 1].t);
      g.ekmin[i] = std::move(tl[i + 1].kmin);
      g.ekmax[i] = std::move(tl[i + 1].kmax);
    }
    p.produced += gemm_produced(g);
  }
  // symmetric plan: blocks with a repeated block index of edge > 1 hold
  // permuted copies to fill after the GEMM
  p.fill_keys.clear();
  if (p.sym)
    for (int64_t k = 0; k < LM.K; ++k)
      for (int q = 1; q < m; ++q)
        if (LM.keys[k * m + q] == LM.keys[k * m + q - 1] && LM.edges[k * m + q] > 1) {
          p.fill_keys.push_back((int32_t)k);
          break;
        }

  // ---- recursion tables ----
  p.part_mask.clear();
  p.part_cnt.clear();
  p.sigma_first.assign(m / 2 + 2, 0);
  std::vector<std::vector<int>> slot_modes;  // per slot: modes (0-based)
  int np = 0;
  for (int sigma = 2; sigma <= m / 2; ++sigma) {
    p.sigma_first[sigma] = np;
    for (auto &parts : partitions_min2(m, sigma)) {
      p.part_cnt.push_back(sigma);
      for (int i = 0; i < 8; ++i) {
        int mask = 0;
        if (i < sigma) {
          std::vector<int> md;
          for (int e : parts[i]) { mask |= 1 << (e - 1); md.push_back(e - 1); }
          slot_modes.push_back(md);
        }
        p.part_mask.push_back(mask);
      }
      ++np;
    }
  }
  p.sigma_first[m / 2 + 1] = np;
  p.nslots = (int32_t)slot_modes.size();
  if (m >= 4) {
    p.sub_rank.resize((size_t)LM.K * p.nslots);
    for (int64_t k = 0; k < LM.K; ++k) {
      const int64_t *key = &LM.keys[k * m];
      for (int s = 0; s < p.nslots; ++s) {
        int64_t sub[16];
        int len = 0;
        for (int q : slot_modes[s]) sub[len++] = key[q];
        p.sub_rank[(size_t)k * p.nslots + s] = (int32_t)multiset_rank(sub, len, p.nbar);
      }
    }
    build_fact_tables(p);
  }
  return "";
}

// factored-recursion tables (recursion_fact.cu): for every order-m key and
// every subset S of modes containing mode 0 with 2 <= |S| <= m-2 (in mask
// order, matching rf::term_mask), the element offsets of the factor blocks
// C_|S|[key|S] and M_{m-|S|}[key|rest] in their packed buffers.
static void build_fact_tables(Plan &p) {
  const int m = p.m;
  p.fact_terms = 0;
  p.term_off.clear();
  p.full_offs.clear();
  p.full_keys.clear();
  p.partial_keys.clear();
  const Layout &LM = p.lay[m];
  for (int64_t k = 0; k < LM.K; ++k) {
    bool full = true;
    for (int q = 0; q < m; ++q) full = full && LM.edges[k * m + q] == p.b;
    (full ? p.full_keys : p.partial_keys).push_back((int32_t)k);
  }
  if (!recursion_fact_supported(m, p.b)) return;
  for (int k = 2; k <= m - 2; ++k)
    if (p.lay[k].offs.back() > INT32_MAX) return;  // offsets kept as int32
  std::vector<int> masks;
  for (int s = 1; s < (1 << m); s += 2) {
    const int c = __builtin_popcount(s);
    if (c >= 2 && c <= m - 2) masks.push_back(s);
  }
  p.fact_terms = (int)masks.size();
  // indexed by position in full_keys (the kernels' work list), so a kernel
  // reads one contiguous row per output block, no key -> table indirection
  p.term_off.resize(p.full_keys.size() * masks.size() * 2);
  p.full_offs.resize(p.full_keys.size());
  for (size_t i = 0; i < p.full_keys.size(); ++i) {
    const int64_t k = p.full_keys[i];
    const int64_t *key = &LM.keys[k * m];
    p.full_offs[i] = LM.offs[k];
    for (size_t t = 0; t < masks.size(); ++t) {
      int64_t a[16], c[16];
      int na = 0, nc = 0;
      for (int q = 0; q < m; ++q) {
        if (masks[t] & (1 << q)) a[na++] = key[q];
        else c[nc++] = key[q];
      }
      p.term_off[(i * masks.size() + t) * 2] = (int32_t)p.lay[na].offs[multiset_rank(a, na, p.nbar)];
      p.term_off[(i * masks.size() + t) * 2 + 1] = (int32_t)p.lay[nc].offs[multiset_rank(c, nc, p.nbar)];
    }
  }
  p.tail_order.clear();
  p.tail_new.clear();
  if (m == 6) {
    p.tail_order.resize(p.full_keys.size());
    std::iota(p.tail_order.begin(), p.tail_order.end(), 0);
    auto key_of = [&](int32_t i) { return &LM.keys[(int64_t)p.full_keys[i] * m]; };
    std::stable_sort(p.tail_order.begin(), p.tail_order.end(), [&](int32_t x, int32_t y) {
      const int64_t *a = key_of(x), *c = key_of(y);
      for (int q = 1; q < m; ++q)
        if (a[q] != c[q]) return a[q] < c[q];
      return a[0] < c[0];
    });
    p.tail_new.assign(p.tail_order.size(), 1);
    for (size_t i = 1; i < p.tail_order.size(); ++i) {
      const int64_t *a = key_of(p.tail_order[i]), *c = key_of(p.tail_order[i - 1]);
      bool same = true;
      for (int q = 1; q < m; ++q) same = same && a[q] == c[q];
      p.tail_new[i] = same ? 0 : 1;
    }
  }
}

template <typename T>
static cudaError_t up(T **dst, const std::vector<T> &src) {
  if (src.empty()) { *dst = nullptr; return cudaSuccess; }
  cudaError_t e = cudaMalloc((void **)dst, src.size() * sizeof(T));
  if (e != cudaSuccess) return e;
  return cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice);
}

std::string upload_plan(Plan &p) {
  cudaError_t e = cudaSuccess;
  for (Gemm &g : p.gemm) {
#define UPG(d, s) if (e == cudaSuccess) e = up(&g.d, g.s)
    UPG(d_rowcols, rowcols);
    UPG(d_colcols, colcols);
    UPG(d_row_keybase, row_keybase);
    UPG(d_row_olin, row_olin);
    UPG(d_row_cstart, row_cstart);
    UPG(d_col_rank, col_rank);
    UPG(d_col_olin, col_olin);
    UPG(d_col_size, col_size);
    UPG(d_tiles, tiles);
    UPG(d_tile_kmin, tile_kmin);
    UPG(d_tile_kmax, tile_kmax);
    for (int i = 0; i < 2; ++i) {
      UPG(d_et[i], et[i]);
      UPG(d_ekmin[i], ekmin[i]);
      UPG(d_ekmax[i], ekmax[i]);
    }
#undef UPG
  }
#define UP(d, s) if (e == cudaSuccess) e = up(&p.d, p.s)
  UP(d_sub_rank, sub_rank);
  UP(d_part_mask, part_mask);
  UP(d_koff, koff);
  UP(d_term_off, term_off);
  UP(d_full_offs, full_offs);
  UP(d_full_keys, full_keys);
  UP(d_partial_keys, partial_keys);
  UP(d_tail_order, tail_order);
  UP(d_tail_new, tail_new);
  UP(d_fill_keys, fill_keys);
#undef UP
  if (e == cudaSuccess) e = up(&p.d_offs, p.lay[p.m].offs);
  if (e == cudaSuccess && p.m >= 1) {
    std::vector<int32_t> k32(p.lay[p.m].keys.begin(), p.lay[p.m].keys.end());
    e = up(&p.d_keys32, k32);
  }
  for (int k = 2; k <= p.m - 2 && e == cudaSuccess; ++k) e = up(&p.d_lower_offs[k], p.lay[k].offs);
  if (e != cudaSuccess) return std::string("plan upload: ") + cudaGetErrorString(e);
  return "";
}

void free_plan(Plan &p) {
  for (Gemm &g : p.gemm) {
    void *gp[] = {g.d_rowcols, g.d_colcols, g.d_row_keybase, g.d_row_olin, g.d_row_cstart,
                  g.d_col_rank, g.d_col_olin, g.d_col_size, g.d_tiles, g.d_tile_kmin, g.d_tile_kmax,
                  g.d_et[0], g.d_ekmin[0], g.d_ekmax[0], g.d_et[1], g.d_ekmin[1], g.d_ekmax[1]};
    for (void *q : gp)
      if (q) cudaFree(q);
  }
  void *ptrs[] = {p.d_offs, p.d_keys32, p.d_sub_rank, p.d_part_mask, p.d_koff, p.d_term_off,
                  p.d_full_offs, p.d_full_keys, p.d_partial_keys, p.d_fill_keys, p.d_tail_order, p.d_tail_new};
  for (void *q : ptrs)
    if (q) cudaFree(q);
  for (auto &q : p.d_lower_offs)
    if (q) { cudaFree(q); q = nullptr; }
}

}  // namespace bcg
