// Near word pairs with their exact distances: the fast form of the near-entry refinement
// (refine.cu) for the symmetric pipeline with a distance table.
//
// refine.cu recomputes a flagged Z entry (a, segment) as the minimum over the segment's
// words b of the exact |a - b|: ~50 x m f32 differences and ~60 KB of rows per entry.  On
// clustered embeddings (the words of a topic close to each other) a few % of the ~1e10
// reverse entries of a step are flagged and that alone takes seconds.  But nearness is a
// property of word PAIRS, and the distance table holds every (query word, vocabulary word)
// distance once: the near pairs are found once per query set, their exact distances
// computed once, and a flagged entry's exact minimum is the minimum over the near pairs
// among its segment's words -- an atomicMin scatter onto the marked entries (common.cuh
// kZMarked), certified equal to the full exact minimum:
//   candidates:  table distance d~(a, b) < 0.75 max(|a|, |b|) + sqrt(m) 2^-22  (scaled;
//                the absolute term covers f16-subnormal rows);
//   near pair of the reverse direction (Z2 row a = query word): exact(a, b) < 0.6 |a|;
//   of the forward direction (Z1 row b = doc word):               exact(a, b) < 0.6 |b|.
// A flagged entry (row a, seg) has d~ < 0.5 |a| at its approximate argmin b_f, so
// exact(a, b_f) < 0.5 |a| + eps < 0.6 |a|: b_f is a near pair and the scatter reaches the
// entry.  Every word of the segment that is not a near pair has exact distance >= 0.6 |a|
// (filtered on the exact value, or no candidate: exact >= 0.75 M - eps >= 0.6 M), above
// the near minimum -- so the near minimum IS the exact segment minimum, bitwise (the same
// exact_sq; min and sqrt are monotone).  eps bounds the Gram form's error: f16 rounding
// 2^-11 (|a| + |b|) plus fp32 accumulation sqrt(4 (m + 2) 2^-21) M (a 4x safety factor
// on a (m + 2) 2^-21 (|a|^2 + |b|^2) bound of d^2): 0.025 M at m = 300, 6x below the
// 0.15 M margin.  An entry no near pair reaches keeps its mark and is recomputed in full
// by refine.cu (finalize), so a candidate list that overflows its capacity -- or a pass
// whose forward direction flagged nothing, where the build is skipped -- costs speed,
// never exactness.
//
// Build (lcrw_near_pairs_build, on the stream, no host sync; all kernels return at once
// when the gate counter -- the forward direction's marked entries -- is 0):
//   candidates  one thread per 16-byte table group (eight keys), warp-aggregated appends
//   exact       one warp per candidate: exact_sq, the two direction tests, per-key counts
//   offsets     CUB inclusive sums of the counts -> two CSRs: reverse keyed by E id u
//               (entries: query-vocabulary row, distance), forward keyed by query-
//               vocabulary row (entries: E id, distance)
//   fill        one thread per candidate
// Zero distances are left out (identical rows are exact zeros already, never flagged).
#include <cub/cub.cuh>

#include "common.cuh"

namespace lcrw {
namespace near {

constexpr int kThreads = 256;

struct Layout {
  size_t hdr, cand, cval, cflag, rev_cnt, rev_off, fwd_cnt, fwd_off, rev_ent, fwd_ent, cub, cub_bytes, total;
};

size_t align256(size_t x) { return (x + 255) / 256 * 256; }

Layout layout(int64_t a_rows, int64_t v_rows, int64_t cap) {
  Layout L;
  size_t cub_bytes = 0;
  const int n_max = (int)(a_rows > v_rows ? a_rows : v_rows);
  cub::DeviceScan::InclusiveSum(nullptr, cub_bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr, n_max > 0 ? n_max : 1);
  L.hdr = 0;
  L.cand = L.hdr + 256;
  L.cval = L.cand + align256((size_t)cap * 8);
  L.cflag = L.cval + align256((size_t)cap * 4);
  L.rev_cnt = L.cflag + align256((size_t)cap);
  L.rev_off = L.rev_cnt + align256((size_t)v_rows * 4);
  L.fwd_cnt = L.rev_off + align256((size_t)(v_rows + 1) * 4);
  L.fwd_off = L.fwd_cnt + align256((size_t)a_rows * 4);
  L.rev_ent = L.fwd_off + align256((size_t)(a_rows + 1) * 4);
  L.fwd_ent = L.rev_ent + align256((size_t)cap * 8);
  L.cub = L.fwd_ent + align256((size_t)cap * 8);
  L.cub_bytes = cub_bytes;
  L.total = L.cub + align256(cub_bytes);
  return L;
}

__device__ __forceinline__ bool gate_closed(const unsigned long long* gate) { return gate && *gate == 0ull; }

// blockIdx.y = table chunk; threads walk its v_rows x 30 groups (contiguous 16-byte loads)
__global__ void __launch_bounds__(kThreads) candidates_kernel(const uint4* __restrict__ T, int64_t row_base,
                                                              int64_t a_rows, int64_t v_rows,
                                                              const float* __restrict__ a_sq,
                                                              const float* __restrict__ v_sq, float delta,
                                                              const unsigned long long* __restrict__ gate,
                                                              unsigned long long* __restrict__ n_cand,
                                                              uint2* __restrict__ cand, int64_t cap) {
  if (gate_closed(gate)) return;
  const int lane = threadIdx.x & 31;
  const int64_t c = blockIdx.y;
  const int64_t groups = v_rows * kTableGroups;
  const uint4* Tc = T + c * groups;
  const int64_t w_chunk = c * kTableChunk;  // table-local row of the chunk's first word
  for (int64_t t0 = (int64_t)blockIdx.x * kThreads; t0 < groups; t0 += (int64_t)gridDim.x * kThreads) {
    const int64_t t = t0 + threadIdx.x;
    uint32_t cm = 0;
    int64_t u = 0, w_base = 0;
    if (t < groups) {
      u = t / kTableGroups;
      w_base = w_chunk + kTableKeysPerGroup * (t - u * kTableGroups);
      const uint4 r = __ldg(Tc + t);
      const uint32_t kw[4] = {r.x, r.y, r.z, r.w};
      const float vs = __ldg(v_sq + u);
#pragma unroll
      for (int j = 0; j < kTableKeysPerGroup; ++j) {
        const int64_t w = w_base + j;
        const uint32_t key = (kw[j >> 1] >> (16 * (j & 1))) & 0xFFFFu;
        if (w < a_rows && key != 0u) {
          const float as = __ldg(a_sq + row_base + w);
          const float thr = kNearCandTau * sqrtf(fmaxf(as, vs)) + delta;
          if (key16_dist(key, key16_base(as)) < thr) cm |= 1u << j;
        }
      }
    }
    // warp-aggregated append: one atomic per warp and step
    const int n = __popc(cm);
    int x = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    const int total = __shfl_sync(0xffffffffu, x, 31);
    if (total == 0) continue;
    unsigned long long base = 0;
    if (lane == 31) base = atomicAdd(n_cand, (unsigned long long)total);
    base = __shfl_sync(0xffffffffu, base, 31);
    unsigned long long pos = base + (unsigned long long)(x - n);
    for (int j = 0; j < kTableKeysPerGroup; ++j)
      if ((cm >> j) & 1u) {
        if (pos < (unsigned long long)cap) cand[pos] = make_uint2((uint32_t)(row_base + w_base + j), (uint32_t)u);
        ++pos;
      }
  }
}

__device__ __forceinline__ bool usable(const unsigned long long* n_cand, int64_t cap, unsigned long long& n) {
  n = *n_cand;
  return n > 0 && n <= (unsigned long long)cap;
}

__global__ void __launch_bounds__(kThreads) exact_kernel(const unsigned long long* __restrict__ n_cand, int64_t cap,
                                                         const uint2* __restrict__ cand, const float* __restrict__ E32,
                                                         int m, const int32_t* __restrict__ a_ids,
                                                         const float* __restrict__ a_sq,
                                                         const float* __restrict__ v_sq,
                                                         const float* __restrict__ scale, float* __restrict__ cval,
                                                         uint8_t* __restrict__ cflag, uint32_t* __restrict__ rev_cnt,
                                                         uint32_t* __restrict__ fwd_cnt) {
  unsigned long long n;
  if (!usable(n_cand, cap, n)) return;
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * kThreads) >> 5;
  const float s0 = __ldg(scale), s2 = s0 * s0;
  const float tau2 = kNearTau * kNearTau;
  for (int64_t j = warp0; j < (int64_t)n; j += n_warps) {
    const uint2 e = cand[j];  // (query-vocabulary row w, E id u)
    const float acc = exact_sq(E32 + (int64_t)__ldg(a_ids + e.x) * m, E32 + (int64_t)e.y * m, m, lane);
    if (lane == 0) {
      const float as = acc * s2;
      const bool rev = acc > 0.f && as < tau2 * __ldg(a_sq + e.x);
      const bool fwd = acc > 0.f && as < tau2 * __ldg(v_sq + e.y);
      cval[j] = sqrtf(acc);
      cflag[j] = (uint8_t)((rev ? 1 : 0) | (fwd ? 2 : 0));
      if (rev) atomicAdd(rev_cnt + e.y, 1u);
      if (fwd) atomicAdd(fwd_cnt + e.x, 1u);
    }
  }
}

__global__ void __launch_bounds__(kThreads) fill_kernel(const unsigned long long* __restrict__ n_cand, int64_t cap,
                                                        const uint2* __restrict__ cand, const float* __restrict__ cval,
                                                        const uint8_t* __restrict__ cflag,
                                                        const uint32_t* __restrict__ rev_off,
                                                        const uint32_t* __restrict__ fwd_off, uint32_t* rev_cur,
                                                        uint32_t* fwd_cur, uint2* __restrict__ rev_ent,
                                                        uint2* __restrict__ fwd_ent) {
  unsigned long long n;
  if (!usable(n_cand, cap, n)) return;
  for (int64_t j = (int64_t)blockIdx.x * kThreads + threadIdx.x; j < (int64_t)n; j += (int64_t)gridDim.x * kThreads) {
    const uint8_t f = cflag[j];
    if (!f) continue;
    const uint2 e = cand[j];
    const uint32_t vb = __float_as_uint(cval[j]);
    if (f & 1) rev_ent[rev_off[e.y] + atomicAdd(rev_cur + e.y, 1u)] = make_uint2(e.x, vb);
    if (f & 2) fwd_ent[fwd_off[e.x] + atomicAdd(fwd_cur + e.x, 1u)] = make_uint2(e.y, vb);
  }
}

// one warp per segment; lane = segment word: its near pairs lower the marked entries
__global__ void __launch_bounds__(kThreads) scatter_kernel(float* __restrict__ Z, int64_t z_panel, int z_shift,
                                                           int64_t n_seg, const int64_t* __restrict__ seg_offsets,
                                                           int64_t seg_base, const int32_t* __restrict__ seg_ids,
                                                           const int32_t* __restrict__ key_map,
                                                           const int32_t* __restrict__ row_map,
                                                           const uint32_t* __restrict__ off,
                                                           const uint2* __restrict__ ent,
                                                           const unsigned long long* __restrict__ n_cand, int64_t cap,
                                                           const unsigned long long* __restrict__ gate) {
  unsigned long long n;
  if (!usable(n_cand, cap, n) || gate_closed(gate)) return;
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * kThreads) >> 5;
  const int64_t zmask = (1ll << z_shift) - 1;
  for (int64_t s = warp0; s < n_seg; s += n_warps) {
    const int64_t t0 = __ldg(seg_offsets + s) - seg_base, t1 = __ldg(seg_offsets + s + 1) - seg_base;
    uint32_t* zs = reinterpret_cast<uint32_t*>(Z + (s >> z_shift) * z_panel + (s & zmask));
    for (int64_t t = t0 + lane; t < t1; t += 32) {
      int32_t key = __ldg(seg_ids + t);
      if (key_map) key = __ldg(key_map + key);
      if (key < 0) continue;
      const uint32_t e1 = __ldg(off + key + 1);
      for (uint32_t x = __ldg(off + key); x < e1; ++x) {
        const uint2 en = __ldg(ent + x);
        const int32_t row = row_map ? __ldg(row_map + en.x) : (int32_t)en.x;
        if (row >= 0) atomicMin(zs + ((int64_t)row << z_shift), kZMarkBit | en.y);
      }
    }
  }
}

int grid_for(int64_t work, int per_block) {
  const int64_t want = ceil_div(work > 0 ? work : 1, per_block);
  const int64_t cap_blocks = (int64_t)sm_count() * 16;
  return (int)(want < cap_blocks ? want : cap_blocks);
}

}  // namespace near
}  // namespace lcrw

using namespace lcrw;

extern "C" {

int lcrw_near_pairs_workspace(int64_t a_rows, int64_t v_rows, int64_t cap, size_t* bytes) {
  LCRW_REQUIRE(a_rows >= 0 && v_rows >= 0 && cap > 0 && cap < (1ll << 32) && bytes,
               "lcrw_near_pairs_workspace: bad arguments (0 < cap < 2^32)");
  LCRW_REQUIRE(a_rows < (1ll << 31) && v_rows < (1ll << 31), "lcrw_near_pairs_workspace: too many rows");
  *bytes = near::layout(a_rows, v_rows, cap).total;
  return LCRW_OK;
}

namespace {
struct NearPtrs {
  unsigned long long* n_cand;
  uint2* cand;
  float* cval;
  uint8_t* cflag;
  uint32_t *rev_cnt, *rev_off, *fwd_cnt, *fwd_off;
  uint2 *rev_ent, *fwd_ent;
  char* cub;
  size_t cub_bytes;
};
NearPtrs near_ptrs(void* ws, int64_t a_rows, int64_t v_rows, int64_t cap) {
  const near::Layout L = near::layout(a_rows, v_rows, cap);
  char* b = static_cast<char*>(ws);
  return NearPtrs{reinterpret_cast<unsigned long long*>(b + L.hdr), reinterpret_cast<uint2*>(b + L.cand),
                  reinterpret_cast<float*>(b + L.cval), reinterpret_cast<uint8_t*>(b + L.cflag),
                  reinterpret_cast<uint32_t*>(b + L.rev_cnt), reinterpret_cast<uint32_t*>(b + L.rev_off),
                  reinterpret_cast<uint32_t*>(b + L.fwd_cnt), reinterpret_cast<uint32_t*>(b + L.fwd_off),
                  reinterpret_cast<uint2*>(b + L.rev_ent), reinterpret_cast<uint2*>(b + L.fwd_ent), b + L.cub,
                  L.cub_bytes};
}
}  // namespace

int lcrw_near_pairs_reset(int64_t a_rows, int64_t v_rows, int64_t cap, void* ws, void* stream) {
  LCRW_REQUIRE(a_rows >= 0 && v_rows >= 0 && cap > 0 && cap < (1ll << 32) && ws, "lcrw_near_pairs_reset: bad arguments");
  const near::Layout L = near::layout(a_rows, v_rows, cap);
  char* b = static_cast<char*>(ws);
  cudaStream_t st = as_stream(stream);
  cudaError_t e;
  // header, counts and the offsets' leading zeros (the offsets' own slots are rewritten)
  if ((e = cudaMemsetAsync(b + L.hdr, 0, 256, st)) != cudaSuccess) return cuda_status(e, "cudaMemsetAsync (near)");
  if ((e = cudaMemsetAsync(b + L.rev_cnt, 0, L.rev_ent - L.rev_cnt, st)) != cudaSuccess)
    return cuda_status(e, "cudaMemsetAsync (near counts)");
  return LCRW_OK;
}

int lcrw_near_pairs_candidates(const void* T, int64_t row_base, int64_t t_rows, int64_t a_rows, int64_t v_rows,
                               const float* a_norms, const float* v_norms, int m, const uint64_t* gate, int64_t cap,
                               void* ws, void* stream) {
  LCRW_REQUIRE(row_base >= 0 && t_rows >= 0 && row_base + t_rows <= a_rows && v_rows >= 0 && m > 0 && cap > 0 &&
                   cap < (1ll << 32),
               "lcrw_near_pairs_candidates: bad shape");
  if (t_rows == 0 || v_rows == 0) return LCRW_OK;
  LCRW_REQUIRE(T && a_norms && v_norms && ws, "lcrw_near_pairs_candidates: null pointer");
  LCRW_REQUIRE(ceil_div(t_rows, kTableChunk) < 65536, "lcrw_near_pairs_candidates: table too large for one launch");
  const NearPtrs P = near_ptrs(ws, a_rows, v_rows, cap);
  cudaStream_t st = as_stream(stream);
  ProfScope prof(st, "near_pairs");
  const int64_t n_chunks = ceil_div(t_rows, kTableChunk);
  const int64_t groups = v_rows * kTableGroups;
  int64_t gx = ceil_div((int64_t)sm_count() * 8, n_chunks);
  if (gx > ceil_div(groups, near::kThreads)) gx = ceil_div(groups, near::kThreads);
  if (gx < 1) gx = 1;
  const float delta = sqrtf((float)m) * 0x1p-22f;
  near::candidates_kernel<<<dim3((unsigned)gx, (unsigned)n_chunks), near::kThreads, 0, st>>>(
      static_cast<const uint4*>(T), row_base, t_rows, v_rows, a_norms, v_norms, delta,
      reinterpret_cast<const unsigned long long*>(gate), P.n_cand, P.cand, cap);
  LCRW_CHECK_LAUNCH("near candidates_kernel");
  return LCRW_OK;
}

int lcrw_near_pairs_finish(int64_t a_rows, int64_t v_rows, const int32_t* a_ids, const float* a_norms,
                           const float* v_norms, const float* E32, int m, const float* scale, int64_t cap, void* ws,
                           void* stream) {
  LCRW_REQUIRE(a_rows >= 0 && v_rows >= 0 && m > 0 && cap > 0 && cap < (1ll << 32), "lcrw_near_pairs_finish: bad shape");
  if (a_rows == 0 || v_rows == 0) return LCRW_OK;
  LCRW_REQUIRE(a_ids && a_norms && v_norms && E32 && scale && ws, "lcrw_near_pairs_finish: null pointer");
  const NearPtrs P = near_ptrs(ws, a_rows, v_rows, cap);
  cudaStream_t st = as_stream(stream);
  ProfScope prof(st, "near_pairs");
  cudaError_t e;
  near::exact_kernel<<<near::grid_for(cap * 32, near::kThreads), near::kThreads, 0, st>>>(
      P.n_cand, cap, P.cand, E32, m, a_ids, a_norms, v_norms, scale, P.cval, P.cflag, P.rev_cnt, P.fwd_cnt);
  LCRW_CHECK_LAUNCH("near exact_kernel");
  size_t cub_bytes = P.cub_bytes;
  if ((e = cub::DeviceScan::InclusiveSum(P.cub, cub_bytes, P.rev_cnt, P.rev_off + 1, (int)v_rows, st)) != cudaSuccess)
    return cuda_status(e, "cub InclusiveSum (near reverse offsets)");
  cub_bytes = P.cub_bytes;
  if ((e = cub::DeviceScan::InclusiveSum(P.cub, cub_bytes, P.fwd_cnt, P.fwd_off + 1, (int)a_rows, st)) != cudaSuccess)
    return cuda_status(e, "cub InclusiveSum (near forward offsets)");
  // the counts become the fill cursors
  if ((e = cudaMemsetAsync(P.rev_cnt, 0, (size_t)v_rows * 4, st)) != cudaSuccess ||
      (e = cudaMemsetAsync(P.fwd_cnt, 0, (size_t)a_rows * 4, st)) != cudaSuccess)
    return cuda_status(e, "cudaMemsetAsync (near cursors)");
  near::fill_kernel<<<near::grid_for(cap, near::kThreads), near::kThreads, 0, st>>>(
      P.n_cand, cap, P.cand, P.cval, P.cflag, P.rev_off, P.fwd_off, P.rev_cnt, P.fwd_cnt, P.rev_ent, P.fwd_ent);
  LCRW_CHECK_LAUNCH("near fill_kernel");
  return LCRW_OK;
}

int lcrw_near_pairs_build(const void* T, int64_t a_rows, int64_t v_rows, const int32_t* a_ids, const float* a_norms,
                          const float* v_norms, const float* E32, int m, const float* scale, const uint64_t* gate,
                          int64_t cap, void* ws, void* stream) {
  int status;
  if ((status = lcrw_near_pairs_reset(a_rows, v_rows, cap, ws, stream))) return status;
  if ((status = lcrw_near_pairs_candidates(T, 0, a_rows, a_rows, v_rows, a_norms, v_norms, m, gate, cap, ws, stream)))
    return status;
  return lcrw_near_pairs_finish(a_rows, v_rows, a_ids, a_norms, v_norms, E32, m, scale, cap, ws, stream);
}

int lcrw_near_scatter(const void* ws, int64_t a_rows, int64_t v_rows, int64_t cap, int direction, float* Z,
                      int64_t z_panel, int z_shift, int64_t n_seg, const int64_t* seg_offsets, int64_t seg_base,
                      const int32_t* seg_ids, const int32_t* key_map, const int32_t* row_map, const uint64_t* gate,
                      void* stream) {
  LCRW_REQUIRE(direction == 0 || direction == 1, "lcrw_near_scatter: direction is 0 (reverse) or 1 (forward)");
  LCRW_REQUIRE(n_seg >= 0 && cap > 0 && z_shift >= 0 && z_shift <= 10, "lcrw_near_scatter: bad shape");
  if (n_seg == 0) return LCRW_OK;
  LCRW_REQUIRE(ws && Z && seg_offsets && seg_ids, "lcrw_near_scatter: null pointer");
  LCRW_REQUIRE(direction == 0 || (key_map && row_map),
               "lcrw_near_scatter: the forward direction maps segment words (E ids) to query-vocabulary rows "
               "(key_map) and E ids to Z rows (row_map)");
  const near::Layout L = near::layout(a_rows, v_rows, cap);
  const char* b = static_cast<const char*>(ws);
  const auto* n_cand = reinterpret_cast<const unsigned long long*>(b + L.hdr);
  const auto* off = reinterpret_cast<const uint32_t*>(b + (direction == 0 ? L.rev_off : L.fwd_off));
  const auto* ent = reinterpret_cast<const uint2*>(b + (direction == 0 ? L.rev_ent : L.fwd_ent));
  cudaStream_t st = as_stream(stream);
  ProfScope prof(st, "near_scatter");
  near::scatter_kernel<<<near::grid_for(n_seg * 32, near::kThreads), near::kThreads, 0, st>>>(
      Z, z_panel, z_shift, n_seg, seg_offsets, seg_base, seg_ids, direction == 0 ? nullptr : key_map,
      direction == 0 ? nullptr : row_map, off, ent, n_cand, cap, reinterpret_cast<const unsigned long long*>(gate));
  LCRW_CHECK_LAUNCH("near scatter_kernel");
  return LCRW_OK;
}

}  // extern "C"
