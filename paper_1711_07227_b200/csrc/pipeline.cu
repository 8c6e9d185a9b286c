// Native driver of the reverse direction (distances.py:263, with the symmetric
// combine of distances.py:264 and the per-query top-k of kernels.py:210-223):
// the resident docs play the queries, the query set is the resident side.
//
// Docs are processed in batches; per batch, on one stream and without host
// synchronisation:
//   gather   T = E_B[words of the batch docs]               (operand rows)
//   plan     segment-end bitmap + column ranges             (segments = docs)
//   phase1   Z2[doc, w] = min_t |E_w - T_t|                 (tcgen05, 32-doc panels)
//   zeros    Z2[doc, w] = 0 where doc holds a word identical to w
//   refine   near Z2 entries (0 < d < tau |E_w|) recomputed exactly from the f32 rows
//            (refine.cu; a scan of the batch's Z2)
//   reverse  D[q, doc] = max(D1, spmm(Xq, Z2)), panel-streaming (query-major D)
// or, with a distance table (table.cu; built once per query set), the first four
// steps are one lcrw_table_min launch (exact zeros are already in the table; it
// marks and lists the near entries), followed by the near-pair scatter (near.cu)
// and the refine step's finalize over the list instead of a scan.
// The loop runs in C++ so a batch costs a handful of launch calls, not Python.
#include <cstdlib>

#include "common.cuh"

namespace lcrw {

namespace {
constexpr int kZShift = 5;  // 32-doc panels: a warp's 32 docs of one word row are one 128-byte line

size_t align256(size_t x) { return (x + 255) / 256 * 256; }

int auto_range_cols(int64_t b_rows, int64_t a_rows) {
  const int64_t n_mtiles = ceil_div(a_rows, 128);
  int64_t want = n_mtiles * b_rows / (8 * (int64_t)sm_count());
  want = (want + 255) / 256 * 256;
  if (want < 1024) want = 1024;
  if (want > 16384) want = 16384;  // a work unit takes two ranges
  return (int)want;
}

constexpr int64_t kRefineCap = 1 << 22;  // refine list entries per batch (overflow -> full scan)

struct Layout {
  size_t T, tn, mask, rs, Z, rlist, rcount, total;
};

Layout layout(int64_t a_rows, int kp, int64_t batch_docs, int64_t max_words) {
  Layout L;
  const int64_t max_ranges = lcrw_plan_ranges(max_words, 1024) + 1;
  L.T = 0;
  L.tn = L.T + align256((size_t)max_words * kp * 2);
  L.mask = L.tn + align256((size_t)max_words * 4);
  L.rs = L.mask + align256((size_t)lcrw_endmask_words(max_words) * 4);
  L.Z = L.rs + align256((size_t)max_ranges * 4);
  const int64_t panels = ceil_div(batch_docs, 1 << kZShift);
  L.rlist = L.Z + align256((size_t)panels * (size_t)(a_rows << kZShift) * 4);
  L.rcount = L.rlist + align256((size_t)kRefineCap * 8);
  L.total = L.rcount + 256;
  return L;
}
}  // namespace
}  // namespace lcrw

using namespace lcrw;

extern "C" {

int lcrw_reverse_workspace(int64_t a_rows, int kp, int64_t batch_docs, int64_t max_batch_words, size_t* bytes) {
  LCRW_REQUIRE(a_rows >= 0 && kp > 0 && batch_docs > 0 && max_batch_words >= 0 && bytes,
               "lcrw_reverse_workspace: bad arguments");
  *bytes = layout(a_rows, kp, batch_docs, max_batch_words).total;
  return LCRW_OK;
}

int lcrw_reverse_pipeline(const uint16_t* A, const float* a_norms, int64_t a_rows, const uint16_t* EhB, int64_t v_rows,
                          int m, int kp,
                          const float* scale, const int64_t* doc_offsets, const int64_t* doc_offsets_host,
                          int64_t n_docs, const int32_t* doc_cols, const int32_t* rep, const int32_t* next,
                          const int32_t* remap, const uint32_t* e_blk, const int64_t* e_tile,
                          int64_t n_q, const float* D1, int64_t d1_ld_panel, float* D, int64_t ld_q, int64_t ld_doc,
                          float* top_d, int64_t* top_i, int k, int64_t id_base, int64_t batch_docs, int range_cols,
                          const void* table, const void* near_ws, int64_t near_cap, int z2_keyed, const float* E32,
                          int dim,
                          const int32_t* a_ids, void* d1_ready, void* ws, size_t ws_bytes, void* stream) {
  LCRW_REQUIRE(n_docs >= 0 && n_q >= 0 && a_rows >= 0, "lcrw_reverse_pipeline: bad shape");
  if (n_docs == 0 || n_q == 0) return LCRW_OK;
  LCRW_REQUIRE(doc_offsets_host && doc_offsets && doc_cols && (rep || table) && ws && (D || top_d) && E32 && a_ids &&
                   dim > 0,
               "lcrw_reverse_pipeline: null pointer");
  LCRW_REQUIRE(batch_docs > 0 && (batch_docs % (1 << kZShift)) == 0,
               "lcrw_reverse_pipeline: batch_docs must be a positive multiple of 32");
  int64_t max_words = 0;
  for (int64_t j0 = 0; !table && j0 < n_docs; j0 += batch_docs) {
    const int64_t j1 = j0 + batch_docs < n_docs ? j0 + batch_docs : n_docs;
    const int64_t w = doc_offsets_host[j1] - doc_offsets_host[j0];
    if (w > max_words) max_words = w;
  }
  const Layout L = layout(a_rows, kp, batch_docs, max_words);
  LCRW_REQUIRE(ws_bytes >= L.total, "lcrw_reverse_pipeline: workspace too small (use lcrw_reverse_workspace)");
  char* base = static_cast<char*>(ws);
  uint16_t* T = reinterpret_cast<uint16_t*>(base + L.T);
  uint32_t* mask = reinterpret_cast<uint32_t*>(base + L.mask);
  int32_t* rs = reinterpret_cast<int32_t*>(base + L.rs);
  float* Z2 = reinterpret_cast<float*>(base + L.Z);
  uint2* rlist = reinterpret_cast<uint2*>(base + L.rlist);
  uint64_t* rcount = reinterpret_cast<uint64_t*>(base + L.rcount);
  const int64_t z_panel = a_rows << kZShift;
  cudaStream_t st = as_stream(stream);
  int status;
  // B operand rows straight from EhB by TMA gather4 (no T copy) when LCRW_GATHER_B=1
  static const bool gather_b = [] {
    const char* e = getenv("LCRW_GATHER_B");
    return e && e[0] == '1';
  }();
  const int64_t v_table = v_rows;
  for (int64_t j0 = 0; j0 < n_docs; j0 += batch_docs) {
    const int64_t j1 = j0 + batch_docs < n_docs ? j0 + batch_docs : n_docs;
    const int64_t nd = j1 - j0;
    const int64_t lo = doc_offsets_host[j0], nw = doc_offsets_host[j1] - lo;
    cudaError_t ce = cudaMemsetAsync(rcount, 0, sizeof(uint64_t), st);
    if (ce != cudaSuccess) return cuda_status(ce, "cudaMemsetAsync (refine count)");
    if (table) {
      // near entries are marked and listed; the near pairs (near.cu) lower them to their exact minima
      if ((status = lcrw_table_min(table, a_rows, v_rows, doc_offsets + j0, lo, nd, doc_cols + lo, scale, Z2,
                                   z_panel, a_norms, rlist, rcount, kRefineCap, stream)))
        return status;
      if (near_ws && (status = lcrw_near_scatter(near_ws, a_rows, v_rows, near_cap, 0, Z2, z_panel, kZShift, nd,
                                                 doc_offsets + j0, lo, doc_cols + lo, nullptr, nullptr, rcount,
                                                 stream)))
        return status;
    } else {
    if (!gather_b && (status = lcrw_gather_rows(EhB, nullptr, kp, doc_cols + lo, nw, T, nullptr, stream)))
      return status;
    const int rc = range_cols > 0 ? range_cols : auto_range_cols(nw, a_rows);
    const int64_t n_ranges = lcrw_plan_ranges(nw, rc);
    if ((status = lcrw_segment_plan(doc_offsets + j0, lo, nd, nw, rc, mask, rs, n_ranges, stream))) return status;
    if ((status = p1::launch(A, a_norms, a_rows, gather_b ? EhB : T, nw, m, kp, doc_offsets + j0, lo, nd, mask, rs,
                             n_ranges, scale, Z2, z_panel, kZShift, st, "phase1_rev",
                             gather_b ? doc_cols + lo : nullptr, v_table, z2_keyed ? 1 /* kZPanelsKey */ : 0)))
      return status;
    if ((status = lcrw_zero_identical(doc_offsets + j0, nd, rep, next, remap, Z2, z_panel, kZShift, stream)))
      return status;
    if (near_ws) {  // mark the near entries for the near-pair scatter
      if ((status = lcrw_refine_near(Z2, z_panel, kZShift, a_rows, nd, doc_offsets + j0, lo, doc_cols + lo, E32,
                                     a_ids, E32, dim, a_norms, scale, nullptr, rcount, 0, z2_keyed ? 1 | 4 : 1,
                                     stream)))
        return status;
      if ((status = lcrw_near_scatter(near_ws, a_rows, v_rows, near_cap, 0, Z2, z_panel, kZShift, nd,
                                      doc_offsets + j0, lo, doc_cols + lo, nullptr, nullptr, rcount, stream)))
        return status;
    }
    }
    // table form: finalize the entries table_min marked and listed (clear the marks the near
    // pairs lowered, recompute the rest); GEMM form: a scan of the batch's Z2 (small next to
    // the GEMM's work) fixing flagged entries -- the same test on the same stored values and
    // bitwise the same results either way
    if ((status = lcrw_refine_near(Z2, z_panel, kZShift, a_rows, nd, doc_offsets + j0, lo, doc_cols + lo, E32, a_ids,
                                   E32, dim, a_norms, scale, table ? rlist : nullptr, rcount, kRefineCap,
                                   (table || near_ws) ? 2 : (z2_keyed ? 0 | 4 : 0), stream)))
      return status;
    if (j0 == 0 && d1_ready) {  // D1 may still be in flight on another stream (forward direction)
      cudaError_t e = cudaStreamWaitEvent(st, reinterpret_cast<cudaEvent_t>(d1_ready), 0);
      if (e != cudaSuccess) return cuda_status(e, "cudaStreamWaitEvent (D1 ready)");
    }
    if ((status = lcrw_reverse_panels(Z2, z_panel, a_rows, nd, j0, e_blk, e_tile, n_q, D1, d1_ld_panel, D, ld_q,
                                      ld_doc, top_d, top_i, k, id_base, stream)))
      return status;
  }
  return LCRW_OK;
}

}  // extern "C"
