/*
 * lcrwmd.h -- C ABI of the B200 (sm_100a) LC-RWMD hot path.
 *
 * The reference (`movers`, /root/reference/pkg/src/movers) is pure Python;
 * its "plugin boundary" is its module API.  Each entry point below replaces
 * the arithmetic of one reference function (file:line cited) and is bound
 * from Python with ctypes (paper_1711_07227_b200/_lib.py); INTEGRATION.md
 * shows the binding.
 *
 * Conventions
 *   - All array pointers are DEVICE pointers owned by the caller; nothing is
 *     allocated or freed here except transient CUB scratch passed in `ws`.
 *   - `stream` is a cudaStream_t (void* to keep CUDA types out of the ABI).
 *     Calls only enqueue work; none synchronises the host unless documented.
 *   - Every function returns an lcrw_status; on failure lcrw_last_error()
 *     returns a thread-local message.  Inputs are never mutated.
 *   - Embedding rows are prepared once as f16 "operand rows" (Xh: rows x kp,
 *     kp = lcrw_padded_dim(m), zero padded) scaled by a power of two held in
 *     a device scalar pair scale[2] = {s, 1/s}; norms are fp32 squared norms
 *     of the rounded scaled rows.  Distances come back unscaled.
 *   - Z ("nearest word distances", distances.py:147-178) is stored in
 *     segment panels: Z[(s >> 3) * z_panel + row * 8 + (s & 7)], z_panel >=
 *     8 * rows.  The same addressing is used for panelled distance outputs.
 */
#ifndef LCRWMD_H_
#define LCRWMD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LCRW_OK = 0,
  LCRW_ERR_INVALID = 1,     /* bad argument (maps to ValueError)            */
  LCRW_ERR_CUDA = 2,        /* CUDA runtime / launch failure (RuntimeError) */
  LCRW_ERR_UNSUPPORTED = 3  /* shape outside what the kernels handle        */
} lcrw_status;

int lcrw_abi_version(void);
const char* lcrw_status_string(int status);
const char* lcrw_last_error(void);
int lcrw_sm_count(int* out);

/* Optional launch profiler (benchmarking): when enabled, instrumented launches
 * (phase1 / phase1_rev / spmm / reverse_panels) are bracketed by CUDA events on
 * their stream; lcrw_profile_get waits for record i and returns its name and
 * elapsed milliseconds. */
int lcrw_profile_reset(int enable);
int64_t lcrw_profile_count(void);
int lcrw_profile_get(int64_t i, char* name, int name_cap, float* ms);

/* ---- embedding preparation (kernels.py:66-69 squared_norms; the f16 operand
 *      rounding replaces the float64 casts of distances.py:161-166) --------
 * Operand rows have K = lcrw_operand_k(m, split) used columns (m or 3m values
 * + 3 norm columns), zero padded to kp = lcrw_padded_dim(K). */
int lcrw_padded_dim(int m);
int lcrw_operand_k(int m, int split);
/* atomically max-accumulates max_r |x_r|^2 over rows x m values into *max_bits (zero it first) */
int lcrw_max_sqnorm(const float* x, int64_t rows, int m, uint32_t* max_bits, void* stream);
/* scale[0] = 2^k with max|x|^2 * 4^k in [2^12, 2^14); scale[1] = 1 / scale[0] */
int lcrw_scale_from_max_sqnorm(const uint32_t* max_bits, float* scale, void* stream);
/* Operand rows of x' = scale * x, hi = f16_rn(x'), lo = f16_rn(x' - hi),
 * n = |rounded row|^2 (fp64) split into three f16 pieces:
 *   layout 0 (A):       [hi, 1, 1, 1]                      K = m + 3
 *   layout 1 (A split): [hi, hi, lo, 1, 1, 1]              K = 3m + 3
 *   layout 2 (B):       [-2hi, n_hi, n_mid, n_lo]          K = m + 3
 *   layout 3 (B split): [-2hi, -2lo, -2hi, n_hi, n_mid, n_lo]  K = 3m + 3
 * so one dot of an A row with a B row is |b|^2 - 2 a.b (split: ~22-bit
 * operands).  norms[r] = n as f32 (may be NULL). */
int lcrw_prepare_rows(const float* X, int64_t rows, int m, int kp, int layout, const float* scale,
                      uint16_t* Xh, float* norms, void* stream);
/* T[i] = Xh[ids[i]], tnorms[i] = norms[ids[i]] if tnorms (distances.py:201 `query_E[cols]`) */
int lcrw_gather_rows(const uint16_t* Xh, const float* norms, int kp, const int32_t* ids, int64_t n,
                     uint16_t* T, float* tnorms, void* stream);

/* ---- exact-identity classes: the reference returns exactly 0 for bitwise
 *      identical vectors (kernels.py:91-92); classes let the GPU reproduce it.
 *      canon[r] = smallest row id with an identical fp32 vector; next[r] links
 *      the members of a class (-1 terminated, starting at the canonical row). */
int lcrw_row_classes_workspace(int64_t rows, size_t* bytes);
int lcrw_row_classes(const float* E, int64_t rows, int m, int32_t* canon, int32_t* next,
                     int64_t* n_dup, uint64_t* sorted_hash, int32_t* sorted_ids, void* ws, size_t ws_bytes,
                     void* stream);
/* rep[i] = canonical E row bitwise equal to Q[i], or -1 */
int lcrw_match_rows(const float* Q, int64_t nq, const float* E, int m, const uint64_t* sorted_hash,
                    const int32_t* sorted_ids, int64_t rows, const int32_t* canon, int32_t* rep, void* stream);

/* ---- vocabulary restriction (corpus.py:405-426) ---- */
int lcrw_restrict_workspace(int64_t n_cols, size_t* bytes);
/* remap[c] = new id or -1; used[0:n_used] ascending; *n_used written on device */
int lcrw_restrict(const int32_t* col_ids, int64_t nnz, int64_t n_cols, int32_t* remap, int32_t* used,
                  int64_t* n_used, void* ws, size_t ws_bytes, void* stream);
/* out[i] = remap[col_ids[i]] (corpus.py:422) */
int lcrw_remap_ids(const int32_t* col_ids, int64_t nnz, const int32_t* remap, int32_t* out, void* stream);

/* ---- Phase 1 (distances.py:147-178 _phase1, kernels.py:72-110) ----------
 * Segment plan: endmask has one bit per B row (set on the last row of each
 * segment), lcrw_endmask_words(n_cols) words (tail padded for the epilogue's
 * 256-column window); range_seg[0..n_ranges] splits the segments into
 * ~range_cols-column ranges that never cut a segment.  Segment s covers B rows
 * [seg_offsets[s] - seg_base, seg_offsets[s+1] - seg_base), so a batch can point
 * into a larger CSR's offsets without rebasing them. */
int64_t lcrw_endmask_words(int64_t n_cols);
int64_t lcrw_plan_ranges(int64_t n_cols, int range_cols);
int lcrw_segment_plan(const int64_t* seg_offsets, int64_t seg_base, int64_t n_seg, int64_t n_cols, int range_cols,
                      uint32_t* endmask, int32_t* range_seg, int64_t n_ranges, void* stream);
/* Z[s, r] = min_{t in segment s} |A_r - B_t| for r < a_rows, s < n_seg, where A
 * rows use layout 0/1 and B rows layout 2/3 of lcrw_prepare_rows, m is their K
 * extent (lcrw_operand_k) and a_norms the A rows' norms:
 * tcgen05 f16 GEMM (TMA-fed, TMEM accumulators) with the Gram expansion and
 * segmented row-min fused into the epilogue.  Z panels are 1 << z_shift
 * segments wide: Z[(s >> z_shift) * z_panel + (r << z_shift) + (s & mask)]. */
int lcrw_phase1(const uint16_t* A, const float* a_norms, int64_t a_rows, const uint16_t* B,
                int64_t b_rows, int m, int kp, const int64_t* seg_offsets,
                int64_t seg_base, int64_t n_seg, const uint32_t* endmask, const int32_t* range_seg,
                int64_t n_ranges, const float* scale, float* Z, int64_t z_panel, int z_shift, void* stream);
/* Exact zeros: for every B row t of segment s whose vector is identical to
 * an A row r (rep[t] / canon / next classes, remap: E id -> A row or -1,
 * NULL = identity), Z[s, r] = 0.  rep is indexed by the raw seg_offsets values. */
int lcrw_zero_identical(const int64_t* seg_offsets, int64_t n_seg, const int32_t* rep,
                        const int32_t* next, const int32_t* remap, float* Z, int64_t z_panel, int z_shift,
                        void* stream);

/* ---- Phase 2 (kernels.py:174-198 spmm/spmv; distances.py:203) -----------
 * out[i, s] = sum_p x[i, p] * Z[s, col[i, p]] in fp64, rounded once to f32,
 * for s < n_seg; out addressed out[i * ld_row + (s >> 3) * ld_panel + (s & 7)].
 * Z in (1 << z_shift)-segment panels, 2 <= z_shift <= 7 (lcrw_phase1 layout):
 * Z[s, w] = Z[(s >> z_shift) * z_panel + (w << z_shift) + (s & mask)].
 * Z may be split into vocabulary blocks of z_block_rows rows (the multi-GPU
 * all-gather of per-rank Phase-1 slices): row w lives at block w / z_block_rows,
 * z_block_stride floats apart; z_block_rows <= 0 means one block. */
int lcrw_spmm(const int64_t* offs, const int32_t* cols, const float* vals, int64_t n_rows, const float* Z,
              int64_t z_panel, int z_shift, int64_t z_block_rows, int64_t z_block_stride, int64_t n_seg, float* out,
              int64_t ld_row, int64_t ld_panel, void* stream);
/* The same product when every Z entry is a distance -- finite, >= 0, zero or normal
 * (lcrw_phase1 / lcrw_refine_near output) -- bitwise equal to lcrw_spmm; the f32 -> f64
 * widening runs on the integer pipe (entries outside that domain give wrong results:
 * use lcrw_spmm for general matrices). */
int lcrw_spmm_dist(const int64_t* offs, const int32_t* cols, const float* vals, int64_t n_rows, const float* Z,
                   int64_t z_panel, int z_shift, int64_t z_block_rows, int64_t z_block_stride, int64_t n_seg,
                   float* out, int64_t ld_row, int64_t ld_panel, void* stream);

/* Reverse direction, panel-streaming form: work item = (32-doc Z2 panel, group
 * of G = lcrw_reverse_panels_group() queries); persistent CTAs stream each
 * panel's word rows through shared memory in T = lcrw_reverse_panels_tile_rows()
 * row tiles and scatter the query nonzeros (the plan below) into fp32
 * per-query accumulators; writes D[q * ld_q + (doc_base + j) * ld_doc] =
 * max(D1, D2) for the batch's docs j < n_docs.  D1 in 8-query panels
 * (d1_ld_panel = 8 * n1).
 * Plan (replaces the word-major traversal of distances.py:203 for the
 * reverse sets): for each query group g and tile t (rows [t*T, t*T+T)) one
 * block of 32-bit words at e_blk + e_tile[g*n_tiles + t] (16-byte aligned,
 * e_tile has n_groups*n_tiles + 1 entries, the last = total words):
 *   W = lcrw_reverse_panels_warps() list ends (entries, cumulative), then the
 *   entries, two words each: ((row - t*T) * 128 << 18 | (q - g*G) * 128, bits of x)
 *   (byte offsets of the Z2 tile row and of the query's accumulator row).
 * Warp w's list is entries [end[w-1], end[w]); a warp owns the queries with
 * (q - g*G) % W == w, so accumulation order is deterministic.  Every list
 * holds a multiple of I = lcrw_reverse_panels_ilp() entries and each aligned
 * group of I entries names I distinct queries; padding entries of warp w's
 * list use query G + w (that warp's scratch row) with weight 0. */
/* The plan above, built on the HOST (plain C++, no device memory): offsets[n_q+1] /
 * cols / vals = the query CSR (E word ids), rank = word id -> query-vocabulary row,
 * T, G, W, I = the lcrw_reverse_panels_* geometry.  Writes words (capacity
 * words_cap >= lcrw_plan_reverse_words_bound(...)), tile_off[n_groups*n_tiles+1]
 * and *n_words.  Output identical to device.plan_query_entries. */
int64_t lcrw_plan_reverse_words_bound(int64_t n_q, int64_t nnz, int64_t a_rows, int T, int G, int W, int I);
int lcrw_plan_reverse(const int64_t* offsets, int64_t n_q, const int32_t* cols, const float* vals,
                      const int32_t* rank, int64_t a_rows, int T, int G, int W, int I, uint32_t* words,
                      int64_t words_cap, int64_t* tile_off, int64_t* n_words);
int lcrw_reverse_panels_tile_rows(void);
int lcrw_reverse_panels_group(void);
int lcrw_reverse_panels_warps(void);
int lcrw_reverse_panels_ilp(void);
int lcrw_reverse_panels(const float* Z2, int64_t z_panel, int64_t a_rows, int64_t n_docs, int64_t doc_base,
                        const uint32_t* e_blk, const int64_t* e_tile, int64_t n_q, const float* D1,
                        int64_t d1_ld_panel, float* D, int64_t ld_q, int64_t ld_doc, float* top_d, int64_t* top_i,
                        int k, int64_t id_base, void* stream);
/* Fused max -> top-k (top_d != NULL, D may be NULL; 1 <= k <= 32): instead of
 * writing D, each CTA keeps the k smallest (distance, id_base + doc_base + j)
 * per query in list slot blockIdx.x: top_d / top_i [n_q][S][k] with S =
 * lcrw_reverse_panels_top_slots(), ascending (distance, id); initialise every
 * entry to (+inf, INT64_MAX) once per query set (the lists carry over between
 * doc batches), then lcrw_topk_segments(top_d, top_i, n_q, S * k, k, ...)
 * gives the per-query top-k of max(D1, D2) without materialising D. */
int lcrw_reverse_panels_top_slots(void);

/* All-pairs symmetric combine (X1 == X2, distances.py:264 with the reverse
 * direction equal to the transposed forward one): D = max(D, D^T) in place for
 * an n x n row-major matrix with row stride ld. */
int lcrw_symmetrize_max(float* D, int64_t n, int64_t ld, void* stream);
/* Sharded all-pairs combine: out[i, j] = max(A[i, j], R[j, i]) for i < rows,
 * j < cols (row strides ldo, lda, ldr; out may equal A).  The caller passes
 * A = the block D1[S_r, S_s] received from rank s, R = this rank's own block
 * D1[S_s, S_r] and out = columns S_s of its output rows. */
int lcrw_max_transposed_into(float* out, int64_t ldo, const float* A, int64_t lda, const float* R, int64_t ldr,
                             int64_t rows, int64_t cols, void* stream);
/* In place: D[i, j] = max(D[i, j], R[j, i]). */
int lcrw_max_transposed(float* D, int64_t ldd, const float* R, int64_t ldr, int64_t rows, int64_t cols,
                        void* stream);

/* Whole reverse direction in one call (distances.py:263-264): docs in batches
 * of batch_docs (multiple of 32); per batch gather -> segment plan ->
 * lcrw_phase1 (32-doc Z2 panels) -> lcrw_zero_identical -> lcrw_reverse_panels,
 * enqueued from C++ on `stream` (EhB has v_rows rows; with LCRW_GATHER_B=1 in
 * the environment the B operand rows are TMA-gathered from EhB by doc_cols
 * inside lcrw_phase1 instead of being copied first).  doc_offsets_host is the host copy of
 * doc_offsets (batch planning); doc_cols are global E ids, rep/next/remap as in
 * lcrw_zero_identical.  Writes D = max(D1, D2) for all docs (see
 * lcrw_reverse_panels).  Workspace from lcrw_reverse_workspace with
 * max_batch_words = max words over batches (0 in table mode).  d1_ready
 * (cudaEvent_t or NULL): the stream waits on it before the first read of D1, so
 * the forward direction can run concurrently on another stream with the reverse
 * Phase 1.  table (NULL = GEMM mode): the packed distance table of
 * lcrw_distance_table for these a_rows query-vocabulary rows and the v_rows E
 * rows; each batch's Z2 is then one lcrw_table_min (gather, plan, phase1 and
 * zeros are skipped; rep, next, remap, EhB may be NULL).  In GEMM mode Z2 is
 * rounded through the table's 16-bit key when z2_keyed != 0, so both modes give the
 * same D (z2_keyed = 0: plain f32 Z2 -- the split-operand precision of m <= 64, where
 * the table form is not chosen).
 * E32 (v_rows x dim f32, unscaled) and a_ids (E id of each A row) feed the
 * exact re-evaluation of near Z2 entries (lcrw_refine_near).  Without near_ws: GEMM
 * form fix-mode scan; table form: lcrw_table_min marks and lists them, finalize over
 * the list.  With near_ws (an lcrw_near_pairs workspace of these a_rows / v_rows and
 * capacity near_cap): the GEMM form marks them (mark scan), lcrw_near_scatter lowers
 * the marked entries of either form, then the finalize mode. */
int lcrw_reverse_workspace(int64_t a_rows, int kp, int64_t batch_docs, int64_t max_batch_words, size_t* bytes);
int lcrw_reverse_pipeline(const uint16_t* A, const float* a_norms, int64_t a_rows, const uint16_t* EhB, int64_t v_rows,
                          int m, int kp,
                          const float* scale, const int64_t* doc_offsets, const int64_t* doc_offsets_host,
                          int64_t n_docs, const int32_t* doc_cols, const int32_t* rep, const int32_t* next,
                          const int32_t* remap, const uint32_t* e_blk, const int64_t* e_tile,
                          int64_t n_q, const float* D1, int64_t d1_ld_panel, float* D, int64_t ld_q, int64_t ld_doc,
                          float* top_d, int64_t* top_i, int k, int64_t id_base, int64_t batch_docs, int range_cols,
                          const void* table, const void* near_ws, int64_t near_cap, int z2_keyed, const float* E32,
                          int dim, const int32_t* a_ids, void* d1_ready, void* ws, size_t ws_bytes, void* stream);

/* ---- distance-table reverse Phase 1 (table.cu) ---------------------------
 * When nnz(X1) >> V, every (w, u) distance of the reverse Phase 1 is needed
 * ~nnz/V times; the table holds each once, as a 16-bit key of the scaled distance
 * relative to its query word w (common.cuh dist_key16: 0 = exact zero, 1 = below
 * 2^e (a near entry), 2..0xFFFE = 2 exponent + 14 mantissa bits over [2^e, 2^(e+4)),
 * round to nearest: relative error <= 2^-15, 0xFFFF = saturated; 2^e <= |w| / 2 <
 * 2^(e+1) from w's scaled squared norm a_norms[w]):
 *   chunk c = w / 256 of 256 query-vocabulary words, per E row u one 512-byte
 *   row at byte ((c * v_rows) + u) * 512 of little-endian uint16 keys, word w of
 *   the chunk at byte 2 (w % 256);  lcrw_table_bytes(a_rows, v_rows) bytes,
 * with exact zeros for identical rows.
 * lcrw_distance_table builds it in one pass: lcrw_phase1 over the a_rows query-
 * vocabulary A rows (lcrw_table_operand_rows(a_rows) == a_rows: no padding) and
 * ALL v_rows E rows (EhB) as singleton segments (seg_offsets = 0..v_rows and its
 * lcrw_segment_plan), storing keys directly (the same entries lcrw_phase1 computes
 * in the GEMM form), then the zeros (canon/next classes of lcrw_row_classes,
 * remap = E id -> A row or -1).
 * lcrw_table_transpose builds the same table from lcrw_phase1's z_shift-7 f32
 * output Tp (unscaled; zeros already applied), the A rows' a_norms and scale
 * (cross-check path).
 * lcrw_table_min: Z2[p * z_panel + w * 32 + (d & 31)] = min over the words u of
 * doc d of T[w, u], decoded and unscaled (32-doc panels, z_panel = 32 * a_rows;
 * docs as lcrw_phase1's segments: doc_offsets[d] - seg_base .. into doc_cols,
 * E ids < v_rows); with refine_list != NULL every near entry (w, d) (lcrw_refine_near's
 * test on the decoded value, a_norms of the A rows) and every saturated one is stored
 * MARKED (all bits set) and
 * appended to the list (*refine_count counts them all, past refine_cap too).  The GEMM form of the reverse pass rounds its Z2 through the
 * same key, so both forms give identical Z2. */
int lcrw_distance_table(const uint16_t* A, const float* a_norms, int64_t a_rows, const uint16_t* EhB, int64_t v_rows,
                        int m, int kp, const int64_t* seg_offsets, const uint32_t* endmask, const int32_t* range_seg,
                        int64_t n_ranges, const float* scale, const int32_t* canon, const int32_t* next,
                        const int32_t* remap, void* T, void* stream);
int lcrw_table_chunk(void);
int64_t lcrw_table_bytes(int64_t a_rows, int64_t v_rows);
int64_t lcrw_table_operand_rows(int64_t a_rows);
int lcrw_table_transpose(const float* Tp, const float* a_norms, int64_t a_rows, int64_t v_rows, const float* scale,
                         void* T, void* stream);
int lcrw_table_min(const void* T, int64_t a_rows, int64_t v_rows, const int64_t* doc_offsets, int64_t seg_base,
                   int64_t n_docs, const int32_t* doc_cols, const float* scale, float* Z2, int64_t z_panel,
                   const float* a_norms, void* refine_list, uint64_t* refine_count, int64_t refine_cap,
                   void* stream);

/* ---- exact re-evaluation of near entries (refine.cu) ---------
 * The Gram expansion's error scales with the operand norms, so an entry whose
 * scaled distance d satisfies 0 < d < tau * |a| (tau = lcrw_refine_tau() = 0.5,
 * |a|^2 = a_norms[row], the A row's scaled squared norm) is recomputed as
 * min over its segment's words b of sqrt(sum_k (A32[a_ids[row]]_k - B32[b]_k)^2)
 * (f32 rows, unscaled, direct differences, fixed order).  Z is lcrw_phase1's
 * panel layout (z_panel, z_shift) of a_rows x n_seg entries; segment s holds
 * B rows seg_ids[seg_offsets[s] - seg_base ..].  list == NULL: every entry is
 * tested (scan).  Otherwise list/count hold the (row, segment) uint32 pairs a
 * producer flagged (lcrw_table_min) and only those are visited -- unless
 * *count > cap, in which case it scans.  mode 0 (fix): flagged entries are
 * recomputed.  mode 1 (mark; scan only): flagged entries are set to all bits
 * (marked) and *count += their number.  mode 2 (finalize): marked entries (sign
 * bit set) that lcrw_near_scatter lowered get the sign bit cleared, those still
 * all bits are recomputed; nothing happens when *count == 0.  All three give the
 * same Z bitwise.  mode | 4 (keyed; fix and mark): Z holds values rounded through the
 * reverse table's 16-bit key (a_norms = its rows' norms): entries at the key's
 * saturation value are flagged too. */
float lcrw_refine_tau(void);
int lcrw_refine_near(float* Z, int64_t z_panel, int z_shift, int64_t a_rows, int64_t n_seg,
                     const int64_t* seg_offsets, int64_t seg_base, const int32_t* seg_ids, const float* A32,
                     const int32_t* a_ids, const float* B32, int m, const float* a_norms, const float* scale,
                     const void* list, uint64_t* count, int64_t cap, int mode, void* stream);

/* ---- near word pairs (near.cu) ---------------------------------
 * The fast form of the refinement when a distance table exists (replaces the
 * per-entry recomputation of kernels.py:72-110 semantics for flagged entries).
 * lcrw_near_pairs_build: from the table T of lcrw_distance_table (a_rows query-
 * vocabulary rows with E ids a_ids and scaled squared norms a_norms; v_rows E rows
 * with scaled squared norms v_norms, f32 rows E32 of width m), the word pairs with
 * table distance < 0.75 max(|a|, |b|) (+ sqrt(m) 2^-22), their exact distances, and
 * two CSRs of the pairs with exact distance < 0.6 |row word|: the reverse one keyed
 * by E id (entries: query-vocabulary row), the forward one keyed by query-vocabulary
 * row (entries: E id).  Enqueued without host sync; skipped (empty lists) when
 * *gate == 0 (gate may be NULL); more than cap candidates leave the lists empty.
 * The first 8 bytes of ws hold the candidate count (uint64).
 * lcrw_near_scatter: for each segment s of Z (lcrw_refine_near's layout) and word t
 * of it, the near pairs of key = seg_ids[t] (forward: key_map[seg_ids[t]], -1 =
 * none) lower each MARKED entry (row, s) -- row = the pair's query-vocabulary row
 * (reverse) or row_map[E id] (forward, -1 = none) -- to the exact distance with
 * the sign bit set (atomicMin); unmarked entries never change.  Nothing happens when
 * *gate == 0 (gate may be NULL).  Then lcrw_refine_near (finalize). */
int lcrw_near_pairs_workspace(int64_t a_rows, int64_t v_rows, int64_t cap, size_t* bytes);
/* lcrw_near_pairs_build = reset + candidates over the whole table + finish.  Without a
 * whole table (the GEMM form: large vocabularies), the candidates come from tables of
 * row slices: lcrw_near_pairs_candidates over a table T of t_rows query-vocabulary rows
 * starting at row row_base (lcrw_distance_table of those rows; its exact zeros are not
 * needed), appending to the list; lcrw_near_pairs_finish then computes the exact
 * distances and the two CSRs. */
int lcrw_near_pairs_reset(int64_t a_rows, int64_t v_rows, int64_t cap, void* ws, void* stream);
int lcrw_near_pairs_candidates(const void* T, int64_t row_base, int64_t t_rows, int64_t a_rows, int64_t v_rows,
                               const float* a_norms, const float* v_norms, int m, const uint64_t* gate, int64_t cap,
                               void* ws, void* stream);
int lcrw_near_pairs_finish(int64_t a_rows, int64_t v_rows, const int32_t* a_ids, const float* a_norms,
                           const float* v_norms, const float* E32, int m, const float* scale, int64_t cap, void* ws,
                           void* stream);
int lcrw_near_pairs_build(const void* T, int64_t a_rows, int64_t v_rows, const int32_t* a_ids, const float* a_norms,
                          const float* v_norms, const float* E32, int m, const float* scale, const uint64_t* gate,
                          int64_t cap, void* ws, void* stream);
int lcrw_near_scatter(const void* ws, int64_t a_rows, int64_t v_rows, int64_t cap, int direction, float* Z,
                      int64_t z_panel, int z_shift, int64_t n_seg, const int64_t* seg_offsets, int64_t seg_base,
                      const int32_t* seg_ids, const int32_t* key_map, const int32_t* row_map, const uint64_t* gate,
                      void* stream);

/* ---- top-k (kernels.py:210-232) ------------------------------------------
 * For each of n_seg segments of seg_len (distance, id) candidates, the k
 * smallest under ascending (distance, id); rows of out hold min(k, seg_len)
 * entries.  k <= 1024 (lcrw_topk_sort handles any k for one segment). */
int lcrw_topk_segments(const float* d, const int64_t* ids, int64_t n_seg, int64_t seg_len, int k,
                       float* out_d, int64_t* out_i, void* stream);
/* per-row top-k of a row-major matrix (row stride ld) with implicit ids id_base + column;
 * rows longer than 16384 with k <= 32 go through per-chunk warp lists and a merge, in a
 * workspace of lcrw_topk_rows_workspace() bytes (0 = none needed, ws may be NULL) */
int lcrw_topk_rows_workspace(int64_t n_rows, int64_t row_len, int k, size_t* bytes);
int lcrw_topk_rows(const float* d, int64_t ld, int64_t n_rows, int64_t row_len, int64_t id_base, int k,
                   float* out_d, int64_t* out_i, void* ws, size_t ws_bytes, void* stream);
int lcrw_topk_sort_workspace(int64_t n, size_t* bytes);
/* full (distance, id) sort of one segment of n candidates; writes the first k */
int lcrw_topk_sort(const float* d, const int64_t* ids, int64_t n, int64_t k, float* out_d, int64_t* out_i,
                   void* ws, size_t ws_bytes, void* stream);
/* topk_select for distances of any numeric dtype (kernels.py:210-223 keeps the caller's
 * dtype: np.lexsort((ids, distances))): element type codes below; the k smallest under
 * ascending (distance, id) with -0 == +0 and NaN after +inf (numpy's order), distances
 * copied to out_d in their own type.  Workspace lcrw_topk_sort_any_workspace(n). */
typedef enum {
  LCRW_F32 = 0, LCRW_F64 = 1, LCRW_F16 = 2,
  LCRW_I8 = 3, LCRW_I16 = 4, LCRW_I32 = 5, LCRW_I64 = 6,
  LCRW_U8 = 7, LCRW_U16 = 8, LCRW_U32 = 9, LCRW_U64 = 10
} lcrw_dtype;
int lcrw_topk_sort_any_workspace(int64_t n, size_t* bytes);
int lcrw_topk_sort_any(const void* d, int dtype, const int64_t* ids, int64_t n, int64_t k, void* out_d,
                       int64_t* out_i, void* ws, size_t ws_bytes, void* stream);

/* ---- reference primitives of the drop-in surface (csrc/prims.cu) ----------
 * Bitwise reproductions of the float64 reference arithmetic (numpy pairwise
 * summation over the contiguous axis, no FMA contraction):
 *   lcrw_squared_norms   kernels.py:66-69   out[r] = sum_i a[r,i]^2 (f64); a f32 or f64 rows x m
 *   lcrw_euclidean_f64   kernels.py:72-110  out[i*ld+j] = sqrt(max(0, (sq_a[i]+sq_b[j]) - 2 a_i.b_j)),
 *                                            stored as f32 (out_dtype LCRW_F32) or f64
 *   lcrw_segmented_min   kernels.py:137-167 minima over the middle axis of an (outer, n, inner)
 *                                            array: segments [seg[s], seg[s+1]) (seg_offsets NULL:
 *                                            one segment = the whole axis: row_min / col_min);
 *                                            np.minimum semantics (NaN propagates), left to right */
int lcrw_squared_norms(const void* a, int dtype, int64_t rows, int64_t m, double* out, void* stream);
int lcrw_euclidean_f64(const double* a, const double* sq_a, int64_t r, const double* b, const double* sq_b, int64_t c,
                       int64_t m, void* out, int out_dtype, int64_t ld, void* stream);
int lcrw_segmented_min(const void* v, int dtype, int64_t outer, int64_t n, int64_t inner, const int64_t* seg_offsets,
                       int64_t n_seg, void* out, void* stream);

/* ---- Exact mover's distance (emd.py:120-211) -------------------------------
 * Batched balanced transport problems, one warp each: successive shortest
 * augmenting paths with node potentials (multi-source Dijkstra over reduced
 * costs clamped at 0, lowest-index ties, tolerance 1e-9), fp64 -- the
 * reference's algorithm.  Problem p: supply[s_off[p] .. s_off[p+1]) (h1),
 * demand[d_off[p] .. d_off[p+1]) (h2), costs row-major h1 x h2 at
 * costs + c_off[p] -- or, with costs == NULL, costs formed from E rows ids1
 * (aligned with supply) and ids2 (aligned with demand) exactly as
 * pairwise_euclidean does (fp64, rounded once to f32; identical rows -> 0).
 * objective[p] = sum(flow * cost); status[p] = 0 ok, 1 no augmenting path with
 * both sides open, 2 no convergence, 3 stopped with supply left because the demand
 * side was exhausted (the reference raises "no augmenting path" there: float32
 * totals differing by > 1e-9; the objective is that of the transported mass).
 * Augmentation stops once either side is exhausted.
 * Optional flow_out (c_off layout) and phi_out (sources at s_off, sinks at
 * s_off[n_problems] + d_off).  c_off is required.  Problems with h1 + h2 <= 128
 * use flow_out as their working storage; pass a buffer of c_off[n_problems]
 * doubles -- with NULL a stream-ordered scratch is allocated per call, which
 * costs a driver allocation each time.  A batch whose largest problem does not fit
 * lcrw_emd_problem_bytes() <= 227 KB of shared memory is solved with the per-problem
 * state in global memory (stream-ordered scratch, launches of <= 4096 problems). */
size_t lcrw_emd_problem_bytes(int h1, int h2);
int lcrw_emd_batch(const double* supply, const int64_t* s_off, const double* demand, const int64_t* d_off,
                   const double* costs, const int64_t* c_off, const float* E, int64_t v, int m, const int32_t* ids1,
                   const int32_t* ids2, int64_t n_problems, int max_h1, int max_h2, double* objective,
                   int32_t* status, double* flow_out, double* phi_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LCRWMD_H_ */
