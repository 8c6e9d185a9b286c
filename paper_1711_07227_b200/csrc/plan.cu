// Host-side plan of the reverse SpMM (lcrw_reverse_panels, include/lcrwmd.h): the query
// set's nonzeros arranged per (query group, Z2 tile, warp) into blocks of 32-bit words.
// The same layout as device.plan_query_entries (the numpy restatement the tests compare
// it with), in native code: it runs on the host every pass while the forward kernels are
// in flight, and with many GPUs (each rank plans the replicated query set while its own
// forward work shrinks) its time is on the critical path.
//
// Per list (g, t, w): the entries (row r, query q, weight x) with q in group g, r in tile
// t, (q - g G) % W == w, ordered by level -- the j-th entry of a query (ascending row) is
// on level j -- and by query inside a level; each level padded to a multiple of I entries
// (padding: scratch query G + w, weight 0), so every aligned group of I names distinct
// queries and each query's terms are summed in ascending row order.
#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"

using namespace lcrw;

extern "C" {

int64_t lcrw_plan_reverse_words_bound(int64_t n_q, int64_t nnz, int64_t a_rows, int T, int G, int W, int I) {
  if (n_q <= 0 || T <= 0 || G <= 0) return 0;
  const int64_t blocks = ((n_q + G - 1) / G) * ((a_rows + T - 1) / T);
  return blocks * (W + 4) + 2 * nnz * I;
}

int lcrw_plan_reverse(const int64_t* offsets, int64_t n_q, const int32_t* cols, const float* vals,
                      const int32_t* rank, int64_t a_rows, int T, int G, int W, int I, uint32_t* words,
                      int64_t words_cap, int64_t* tile_off, int64_t* n_words) {
  LCRW_REQUIRE(offsets && cols && vals && rank && words && tile_off && n_words, "lcrw_plan_reverse: null pointer");
  LCRW_REQUIRE(n_q >= 0 && a_rows >= 0 && T > 0 && T <= 128 && G > 0 && G <= 1024 && W > 0 && I > 0,
               "lcrw_plan_reverse: plan encoding holds rows < 128 and queries <= 1024");
  const int64_t n_tiles = (a_rows + T - 1) / T;
  const int64_t n_groups = (n_q + G - 1) / G;
  const int64_t n_blocks = n_groups * n_tiles;
  const int64_t n_lists = n_blocks * W;
  const int64_t nnz = n_q ? offsets[n_q] : 0;
  struct Ent {
    int32_t ql, rl, level;
    uint32_t x;
  };
  // bucket the nonzeros by list (counting sort, stable in (query, CSR position))
  std::vector<int64_t> list_of(nnz);
  std::vector<int64_t> cnt(n_lists + 1, 0);
  for (int64_t q = 0; q < n_q; ++q) {
    const int64_t g = q / G, ql = q % G;
    for (int64_t e = offsets[q]; e < offsets[q + 1]; ++e) {
      const int64_t r = rank[cols[e]];
      const int64_t key = (g * n_tiles + r / T) * W + ql % W;
      list_of[e] = key;
      ++cnt[key + 1];
    }
  }
  for (int64_t i = 0; i < n_lists; ++i) cnt[i + 1] += cnt[i];
  std::vector<Ent> ent(nnz);
  {
    std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
    for (int64_t q = 0; q < n_q; ++q)
      for (int64_t e = offsets[q]; e < offsets[q + 1]; ++e) {
        Ent v;
        v.ql = (int32_t)(q % G);
        v.rl = (int32_t)(rank[cols[e]] % T);
        v.level = 0;
        std::memcpy(&v.x, vals + e, 4);
        ent[fill[list_of[e]]++] = v;
      }
  }
  // per list: (query, row) order -> levels -> (level, query) order; padded list lengths
  std::vector<int64_t> padded(n_lists, 0);
  for (int64_t l = 0; l < n_lists; ++l) {
    Ent* b = ent.data() + cnt[l];
    Ent* e = ent.data() + cnt[l + 1];
    std::sort(b, e, [](const Ent& a, const Ent& c) { return a.ql != c.ql ? a.ql < c.ql : a.rl < c.rl; });
    for (Ent* p = b; p < e; ++p) p->level = (p > b && (p - 1)->ql == p->ql) ? (p - 1)->level + 1 : 0;
    std::sort(b, e, [](const Ent& a, const Ent& c) { return a.level != c.level ? a.level < c.level : a.ql < c.ql; });
    int64_t len = 0;
    for (Ent* p = b; p < e;) {
      Ent* q = p;
      while (q < e && q->level == p->level) ++q;
      len += (q - p + I - 1) / I * I;
      p = q;
    }
    padded[l] = len;
  }
  // block offsets: W list ends + 2 words per (padded) entry, 16-byte aligned blocks
  tile_off[0] = 0;
  for (int64_t B = 0; B < n_blocks; ++B) {
    int64_t ends = 0;
    for (int w = 0; w < W; ++w) ends += padded[B * W + w];
    const int64_t bw = (W + 2 * ends + 3) / 4 * 4;
    tile_off[B + 1] = tile_off[B] + bw;
  }
  *n_words = tile_off[n_blocks];
  LCRW_REQUIRE(*n_words <= words_cap, "lcrw_plan_reverse: words buffer too small (lcrw_plan_reverse_words_bound)");
  std::memset(words, 0, (size_t)*n_words * 4);
  for (int64_t B = 0; B < n_blocks; ++B) {
    uint32_t* blk = words + tile_off[B];
    int64_t end = 0;
    uint32_t* slot = blk + W;
    for (int w = 0; w < W; ++w) {
      const int64_t l = B * W + w;
      end += padded[l];
      blk[w] = (uint32_t)end;
      const uint32_t pad = (uint32_t)(G + w) * 128u;
      const Ent* b = ent.data() + cnt[l];
      const Ent* e = ent.data() + cnt[l + 1];
      for (const Ent* p = b; p < e;) {
        const Ent* q = p;
        while (q < e && q->level == p->level) ++q;
        const int64_t n = q - p, np = (n + I - 1) / I * I;
        for (int64_t i = 0; i < np; ++i, slot += 2) {
          if (i < n) {
            slot[0] = (((uint32_t)p[i].rl * 128u) << 18) | ((uint32_t)p[i].ql * 128u);
            slot[1] = p[i].x;
          } else {
            slot[0] = pad;
            slot[1] = 0u;
          }
        }
        p = q;
      }
    }
  }
  return LCRW_OK;
}

}  // extern "C"
