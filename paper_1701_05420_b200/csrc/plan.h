// Host-built index tables for one (n, m, b).  See DESIGN.md "Data layout in HBM".
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace bcg {

// The reference's _block_layout for one order (bc/_engines.py:46-54).
struct Layout {
  int order = 0;
  int64_t K = 0;                 // blocks = C(nbar + order - 1, order)
  std::vector<int64_t> keys;     // K x order, 1-based sorted keys, lexicographic
  std::vector<int64_t> col0;     // K x order, (j - 1) * b
  std::vector<int64_t> edges;    // K x order
  std::vector<int64_t> offs;     // K + 1 prefix sums of block sizes
};

// Moment CTA tile (rows = left Khatri-Rao columns, cols = right ones).
constexpr int kTM = 64;
constexpr int kTN = 64;

struct Tile {
  int32_t row0, col0;
};

// One staircase GEMM of the order-m moment: rows = left h-tuples (grouped by
// their last entry v), cols = right r-tuples (lexicographic); row group v's
// valid columns are the suffix from cs(max(v, tcol)).
struct Gemm {
  int h = 0, r = 0;
  int tm = kTM, tn = kTN;               // CTA tile
  int64_t R = 0, C = 0;                 // left rows, right cols
  std::vector<int16_t> rowcols;         // R x h X-column per mode
  std::vector<int16_t> colcols;         // C x r
  std::vector<int32_t> row_keybase;     // key index of (L, R) = row_keybase + col_rank
  std::vector<int32_t> row_olin;        // within-block linear offset of L's modes
  std::vector<int32_t> row_cstart;      // first valid col of the row's group
  std::vector<int32_t> col_rank;        // lexicographic rank of R among r-tuples
  std::vector<int32_t> col_olin;        // within-block offset of R's modes
  std::vector<int32_t> col_size;        // |R| = prod edges(R)
  std::vector<Tile> tiles;
  std::vector<int32_t> tile_kmin, tile_kmax;  // key range a tile touches
  // band-edge tiles: a band's tail is covered by narrower tiles of width
  // ew[0] = tn/2 and ew[1] = tn/4 (0 = not a compiled shape) -- the staircase
  // overhang; et[i] / ekmin[i] / ekmax[i] as tiles / tile_kmin / tile_kmax
  int ew[2] = {0, 0};
  std::vector<Tile> et[2];
  std::vector<int32_t> ekmin[2], ekmax[2];
  // device copies
  int16_t *d_rowcols = nullptr, *d_colcols = nullptr;
  int32_t *d_row_keybase = nullptr, *d_row_olin = nullptr, *d_row_cstart = nullptr;
  int32_t *d_col_rank = nullptr, *d_col_olin = nullptr, *d_col_size = nullptr;
  Tile *d_tiles = nullptr;
  int32_t *d_tile_kmin = nullptr, *d_tile_kmax = nullptr;
  Tile *d_et[2] = {nullptr, nullptr};
  int32_t *d_ekmin[2] = {nullptr, nullptr}, *d_ekmax[2] = {nullptr, nullptr};
};

struct Plan {
  int64_t n = 0;
  int variant = 0;          // moment kernel variant (0: the DMMA kernel)
  // symmetric plan (default): within every run of equal block indices of a
  // GEMM row (left) or column (right) tuple only the in-block offsets with
  // non-decreasing digits are produced; the permuted copies are filled from
  // them afterwards (k_sym_fill).  false: every stored element is produced
  // directly (the reference's per-element semantics, bc/_core.pyx:60-123).
  bool sym = true;
  int m = 0, b = 0;
  int64_t nbar = 0;
  std::vector<Layout> lay;  // index = order, 0..m (0 unused)

  // --- moment GEMM(s) of order m ---
  // One GEMM with h = m/2, or for odd m the hybrid split: keys with
  // key[h] >= split_T in the (h | r) GEMM, keys with key[h] < split_T in the
  // (h+1 | r-1) GEMM (both staircases nearly rectangular, K2).
  std::vector<Gemm> gemm;
  int split_T = 0;                      // 0: single GEMM
  std::vector<int64_t> koff;           // key -> output offset of its block
  int64_t S_out = 0;                   // output elements (S_m)
  int64_t produced = 0;                // elements the GEMMs produce (S_m unless sym)
  // sym: blocks whose key repeats a block index (edge > 1) -- the fill list
  std::vector<int32_t> fill_keys;

  // --- recursion (order m) ---
  // partition table: for sigma = 2..m/2, partitions in reference order
  // (bc/partitions.py:63-98).  part_mask[p * 8 + i] = bitmask of modes (0-based)
  // of part i of partition p; part_cnt[p] = sigma; sigma_first[s] = first p.
  std::vector<int32_t> part_mask;
  std::vector<int32_t> part_cnt;
  std::vector<int32_t> sigma_first;     // size m/2 + 2, sigma_first[sigma]
  int32_t nslots = 0;                   // total (partition, part) pairs
  std::vector<int32_t> sub_rank;        // K_m x nslots lower-block index per slot
  // factored recursion (recursion_fact.cu): terms S containing mode 0
  int fact_terms = 0;                   // 0: not supported for (m, b)
  std::vector<int32_t> term_off;        // full blocks x terms x 2 factor-block element offsets
  std::vector<int64_t> full_offs;       // M_m element offset of each full block
  std::vector<int32_t> full_keys, partial_keys;  // blocks with all edges == b / the rest
  // order-6 streamed recursion (recursion_stream.cu): work-list positions
  // sorted by the key's modes 1..5 (blocks sharing them share every second
  // factor), then by mode 0
  std::vector<int32_t> tail_order;
  std::vector<int32_t> tail_new;        // per position of tail_order: 1 = the tail differs from the previous position's

  // --- device copies ---
  int64_t *d_offs = nullptr;           // offs of order m
  int32_t *d_keys32 = nullptr;          // K_m x m keys (1-based)
  int32_t *d_sub_rank = nullptr;
  int32_t *d_part_mask = nullptr;
  int64_t *d_koff = nullptr;
  int32_t *d_term_off = nullptr;
  int64_t *d_full_offs = nullptr;
  int32_t *d_full_keys = nullptr, *d_partial_keys = nullptr;
  int32_t *d_tail_order = nullptr, *d_tail_new = nullptr;
  int32_t *d_fill_keys = nullptr;
  int64_t *d_lower_offs[16] = {nullptr};  // offs of orders 2..m-2
};

// Builders (plan.cu).
std::string build_plan(int64_t n, int m, int b, Plan &p, int variant = -1, bool sym = true);
int default_variant();
std::string upload_plan(Plan &p);
void free_plan(Plan &p);
int64_t multiset_rank(const int64_t *key, int k, int64_t nbar);
std::vector<std::vector<std::vector<int>>> partitions_min2(int m, int sigma);

}  // namespace bcg
