// Distance-table form of the reverse Phase 1 (distances.py:147-178 with the
// resident docs as "queries", distances.py:263).
//
// The reverse direction needs Z2[w, doc] = min_{u in doc} |E2_w - E_u| for every
// query-vocabulary word w and every resident doc.  The GEMM form recomputes
// |E2_w - E_u| once per OCCURRENCE of u (nnz(X1) columns); when the vocabulary is
// much smaller than nnz(X1) every pair (w, u) is recomputed ~nnz/V times (~500x at
// BASELINE configs[1]).  The table form computes each pair once with the same
// Phase-1 kernel (same operands, same roles: A = E2 rows, B = E rows as singleton
// segments, so every entry is bitwise the value the GEMM form produces), applies
// the exact zeros, and stores it as 256-word chunks [chunk][u][256 w] of 16-bit keys
// (one 512-byte row per vocabulary word, common.cuh); each doc's Z2 column is then a
// min over its words' rows: 512-byte gathers from an L2-resident 51 MB chunk
// (V = 100k), L2-bandwidth bound instead of tensor bound.
#include "common.cuh"

namespace lcrw {
namespace tbl {


// L2 policies: the table chunk is re-read by every doc (evict_last); doc word ids
// and Z2 stores stream through once (evict_first), so they do not push the chunk out
__device__ __forceinline__ uint64_t l2_policy_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint4 ld_keep_u4(const uint4* ptr, uint64_t pol) {
  uint4 v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
      : "l"(ptr), "l"(pol));
  return v;
}
__device__ __forceinline__ int ld_stream(const int32_t* ptr, uint64_t pol) {
  int v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(ptr), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_stream(float* ptr, float v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(ptr), "f"(v), "l"(pol) : "memory");
}

constexpr int kChunk = kTableChunk;  // query-vocabulary words per table chunk (512-byte rows)
constexpr int kPanelDocs = 32;       // Z2 panel width (lcrw_reverse_panels layout)
// smem positions of the chunk's words: one pad slot per 32 words, so a lane's eight
// consecutive words (8 l + j) fall in distinct banks across the warp for every j, and an
// odd row stride keeps the per-word reads of 32 docs conflict-free too
__device__ __forceinline__ int tpos(int w) { return w + (w >> 5); }
constexpr int kTilePos = kChunk + kChunk / 32;  // 264 positions per row
constexpr int kTileStride = kTilePos + 1;       // 265 (odd)
#ifndef LCRW_TBL_MINB
#define LCRW_TBL_MINB 5  // 5 CTAs (40 warps) per SM: <= 48 registers
#endif

// Sets word w's key in row u (cross-check and exact-zero paths; the build writes rows
// straight from the Phase-1 epilogue)
__device__ __forceinline__ void store_key(uint8_t* T, int64_t v_rows, int64_t w, int64_t u, uint32_t key) {
  *reinterpret_cast<uint16_t*>(T + ((w / kChunk) * v_rows + u) * kTableRowBytes + (w % kChunk) * 2) = (uint16_t)key;
}

// Cross-check path: T'[(u >> 7) * zp + (w << 7) + (u & 127)] (f32 segment panels of lcrw_phase1,
// z_shift 7, zp = a_rows * 128, unscaled distances) -> the table (keys of the scaled values).
__global__ void __launch_bounds__(256) transpose_kernel(const float* __restrict__ Tp,
                                                        const float* __restrict__ a_norms, int64_t a_rows,
                                                        int64_t v_rows, const float* __restrict__ scale,
                                                        uint8_t* __restrict__ T) {
  __shared__ float t[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t u0 = (int64_t)blockIdx.x * 32, w0 = (int64_t)blockIdx.y * 32;
  const int64_t zp = a_rows * 128;  // z_shift-7 segment panels
  const float s = scale[0];
  for (int y = ty; y < 32; y += 8) {  // source rows w0 + y, columns u0 + tx (contiguous in u)
    const int64_t w = w0 + y, u = u0 + tx;
    t[y][tx] = (w < a_rows && u < v_rows) ? Tp[(u >> 7) * zp + (w << 7) + (u & 127)] : 0.f;
  }
  __syncthreads();
  for (int y = ty; y < 32; y += 8) {  // destination rows u0 + y, words w0 + tx
    const int64_t u = u0 + y, w = w0 + tx;
    if (u < v_rows && w < a_rows) store_key(T, v_rows, w, u, dist_key16(t[tx][y] * s, key16_base(a_norms[w])));
  }
}

// Exact zeros (kernels.py:91-92, as lcrw_zero_identical): key 0 for every query-vocabulary
// row w whose E row is bitwise identical to E row u (class chain of canon[u]).
__global__ void table_zeros_kernel(const int32_t* __restrict__ canon, const int32_t* __restrict__ next,
                                   const int32_t* __restrict__ remap, int64_t v_rows, uint8_t* __restrict__ T) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < v_rows;
       u += (int64_t)gridDim.x * blockDim.x) {
    for (int32_t g = canon[u]; g >= 0; g = next[g]) {
      const int32_t r = remap[g];
      if (r >= 0) store_key(T, v_rows, r, u, 0u);
    }
  }
}

// One CTA per work unit (chunk c, 32-doc panel p), panels fastest, so the CTAs in flight
// share one L2-resident chunk (v_rows x 512 B: 51 MB at V = 100k); 5 CTAs per SM.  (A
// persistent loop over units measured 2.6x slower: CTAs drift apart and the chunks in
// flight no longer fit L2.)  Warp j takes docs j, j+8, j+16, j+24.  Per 32 doc words the
// warp stages the word ids in its smem slot and broadcasts them four at a time (one
// LDS.128 wavefront per 4 rows -- a SHFL per row shares the L1TEX data pipe with the
// table loads and measured 10 % slower); lane l owns words 8l..8l+7 of the chunk: per doc
// word, one 16-byte load of their eight 16-bit keys (the warp reads the 512-byte row
// once: 256 distances, 2 bytes each), 4 rows in flight, the minima as four SIMD 16-bit
// minima (__vminu2).  The 32 x 256 result is decoded (each word's key range), unscaled,
// staged in smem (one pad slot per 32 words, odd row stride 265: conflict-free both ways)
// and written as 256 coalesced
// 128-byte Z2 rows: Z2[p * z_panel + w * 32 + doc].
__global__ void __launch_bounds__(256, LCRW_TBL_MINB) table_min_kernel(const uint8_t* __restrict__ T, int64_t v_rows, int64_t a_rows,
                                                        const int64_t* __restrict__ doc_offsets, int64_t seg_base,
                                                        int64_t n_docs, const int32_t* __restrict__ cols,
                                                        const float* __restrict__ scale, float* __restrict__ Z2,
                                                        int64_t z_panel, int64_t panels,
                                                        const float* __restrict__ a_norms, RefineSink sink) {
  __shared__ float tile[kPanelDocs * kTileStride];
  __shared__ float wsq[kChunk];               // the chunk words' scaled squared norms (refine test)
  __shared__ uint32_t kb[kTilePos];           // the chunk words' key ranges (key16_base), at tpos(w)
  __shared__ __align__(16) int ids_s[8][32];  // per-warp word ids of the current 32-word block
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t keep = l2_policy_last(), stream = l2_policy_first();
  const float inv_scale = __ldg(scale + 1);
  const int64_t c = blockIdx.x / panels, p = blockIdx.x - c * panels;
  {
    const int q = threadIdx.x;  // 256 threads = the chunk's 256 words
    const float a_sq = c * kChunk + q < a_rows ? __ldg(a_norms + c * kChunk + q) : 0.f;
    wsq[q] = a_sq;
    kb[tpos(q)] = key16_base(a_sq);
  }
  __syncthreads();
  const uint4* Tc = reinterpret_cast<const uint4*>(T + c * v_rows * kTableRowBytes) + lane;
  for (int dd = warp; dd < kPanelDocs; dd += 8) {
    const int64_t d = p * kPanelDocs + dd;
    uint4 k = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
    if (d < n_docs) {
      const int64_t b = __ldg(doc_offsets + d) - seg_base, e = __ldg(doc_offsets + d + 1) - seg_base;
      for (int64_t j0 = b; j0 < e; j0 += 32) {
        const int n = e - j0 < 32 ? (int)(e - j0) : 32;
        __syncwarp();
        ids_s[warp][lane] = lane < n ? ld_stream(cols + j0 + lane, stream) : 0;
        __syncwarp();
        const int4* q4 = reinterpret_cast<const int4*>(ids_s[warp]);
        auto min8 = [&](const uint4 r) {
          k.x = __vminu2(k.x, r.x);
          k.y = __vminu2(k.y, r.y);
          k.z = __vminu2(k.z, r.z);
          k.w = __vminu2(k.w, r.w);
        };
        int j = 0;
#pragma unroll 1
        for (; j + 4 <= n; j += 4) {
          const int4 u4 = q4[j >> 2];
          const uint4 r0 = ld_keep_u4(Tc + (int64_t)u4.x * (kTableRowBytes / 16), keep);
          const uint4 r1 = ld_keep_u4(Tc + (int64_t)u4.y * (kTableRowBytes / 16), keep);
          const uint4 r2 = ld_keep_u4(Tc + (int64_t)u4.z * (kTableRowBytes / 16), keep);
          const uint4 r3 = ld_keep_u4(Tc + (int64_t)u4.w * (kTableRowBytes / 16), keep);
          min8(r0);
          min8(r1);
          min8(r2);
          min8(r3);
        }
        for (; j < n; ++j) min8(ld_keep_u4(Tc + (int64_t)ids_s[warp][j] * (kTableRowBytes / 16), keep));
      }
    }
    // the lane's words 8 lane + j sit at tpos(8 lane + j) = 8 lane + lane / 4 + j
    const int pos = kTableKeysPerGroup * lane + (lane >> 2);
    float* trow = tile + dd * kTileStride + pos;
    const uint32_t* kq = kb + pos;
    const uint32_t kw[4] = {k.x, k.y, k.z, k.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      trow[2 * i] = key16_dist(kw[i] & 0xFFFFu, kq[2 * i]) * inv_scale;
      trow[2 * i + 1] = key16_dist(kw[i] >> 16, kq[2 * i + 1]) * inv_scale;
    }
  }
  __syncthreads();
  // the chunk's largest squared norm and smallest saturation value: an entry at or above
  // tau * max|a| and below the smallest saturation value needs no per-word test
  float wsq_max = 0.f, sat_min = __int_as_float(0x7f800000);
  if (sink.list) {
    for (int q = lane; q < kChunk; q += 32) {
      if (c * kChunk + q < a_rows) {
        wsq_max = fmaxf(wsq_max, wsq[q]);
        sat_min = fminf(sat_min, key16_sat(kb[tpos(q)]));
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      wsq_max = fmaxf(wsq_max, __shfl_xor_sync(0xffffffffu, wsq_max, o));
      sat_min = fminf(sat_min, __shfl_xor_sync(0xffffffffu, sat_min, o));
    }
  }
  const float s0 = __ldg(scale);
  float* zp = Z2 + p * z_panel;
  const int64_t w0 = c * kChunk;
  const bool doc_ok = p * kPanelDocs + lane < n_docs;
  const float* trow = tile + lane * kTileStride;
  // near entries (lcrw_refine_near's scan test on the value) and saturated keys are stored
  // marked (kZMarked); lcrw_near_scatter / lcrw_refine_near (finalize) replace them
  auto is_near = [&](int q, float v) {
    const float ds = v * s0;
    return sink.list && doc_ok &&
           ((ds * ds < kRefineTau * kRefineTau * wsq_max && refine_flag(ds, wsq[q], kRefineTau * kRefineTau)) ||
            (ds >= sat_min && ds >= key16_sat(kb[tpos(q)])));
  };
  uint32_t n_near = 0;
  for (int q = warp; q < kChunk; q += 8) {  // lane = doc; word q of the chunk
    if (w0 + q < a_rows) {
      const float v = trow[tpos(q)];
      const bool near = is_near(q, v);
      st_stream(zp + (w0 + q) * kPanelDocs + lane, near ? __uint_as_float(kZMarked) : v, stream);
      n_near += __popc(__ballot_sync(0xffffffffu, near));
    }
  }
  if (!sink.list) return;
  // the refine list: one global atomic per CTA (a per-entry counter serialises on clustered
  // data), then the entries -- only while the list has room
  __shared__ uint32_t warp_near[8];
  __shared__ unsigned long long cta_base;
  if (lane == 0) warp_near[warp] = n_near;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t total = 0;
    for (int w = 0; w < 8; ++w) total += warp_near[w];
    cta_base = total ? atomicAdd(sink.count, (unsigned long long)total) : ~0ull;
  }
  __syncthreads();
  if (cta_base >= (unsigned long long)sink.cap) return;
  unsigned long long pos = cta_base;
  for (int w = 0; w < warp; ++w) pos += warp_near[w];
  for (int q = warp; q < kChunk && n_near; q += 8) {
    if (w0 + q < a_rows) {
      const bool near = is_near(q, trow[tpos(q)]);
      const uint32_t ballot = __ballot_sync(0xffffffffu, near);
      const unsigned long long mine = pos + __popc(ballot & ((1u << lane) - 1u));
      if (near && mine < (unsigned long long)sink.cap)
        sink.list[mine] = make_uint2((uint32_t)(w0 + q), (uint32_t)(p * kPanelDocs + lane));
      pos += __popc(ballot);
    }
  }
}

}  // namespace tbl
}  // namespace lcrw

using namespace lcrw;

extern "C" {

int lcrw_table_chunk(void) { return tbl::kChunk; }

int64_t lcrw_table_bytes(int64_t a_rows, int64_t v_rows) {
  return ceil_div(a_rows, tbl::kChunk) * v_rows * kTableRowBytes;
}

int64_t lcrw_table_operand_rows(int64_t a_rows) { return a_rows; }

int lcrw_distance_table(const uint16_t* A, const float* a_norms, int64_t a_rows, const uint16_t* EhB, int64_t v_rows,
                        int m, int kp, const int64_t* seg_offsets, const uint32_t* endmask, const int32_t* range_seg,
                        int64_t n_ranges, const float* scale, const int32_t* canon, const int32_t* next,
                        const int32_t* remap, void* T, void* stream) {
  LCRW_REQUIRE(a_rows >= 0 && v_rows >= 0, "lcrw_distance_table: bad shape");
  if (a_rows == 0 || v_rows == 0) return LCRW_OK;
  LCRW_REQUIRE(canon && next && remap && T, "lcrw_distance_table: null pointer");
  cudaStream_t st = as_stream(stream);
  // (the build writes every key of the last chunk: rows past a_rows hold unused values)
  int status = p1::launch(A, a_norms, a_rows, EhB, v_rows, m, kp, seg_offsets, 0, v_rows, endmask, range_seg,
                          n_ranges, scale, static_cast<float*>(T), v_rows * kTableRowBytes, 7, st, "table_build",
                          nullptr, 0, 2 /* kZTable */);
  if (status) return status;
  const int64_t blocks = ceil_div(v_rows, 256);
  tbl::table_zeros_kernel<<<(unsigned)(blocks < 4096 ? blocks : 4096), 256, 0, st>>>(canon, next, remap, v_rows,
                                                                                     static_cast<uint8_t*>(T));
  LCRW_CHECK_LAUNCH("table_zeros_kernel");
  return LCRW_OK;
}

int lcrw_table_transpose(const float* Tp, const float* a_norms, int64_t a_rows, int64_t v_rows, const float* scale,
                         void* T, void* stream) {
  LCRW_REQUIRE(a_rows >= 0 && v_rows >= 0, "lcrw_table_transpose: bad shape");
  if (a_rows == 0 || v_rows == 0) return LCRW_OK;
  LCRW_REQUIRE(Tp && a_norms && T && scale, "lcrw_table_transpose: null pointer");
  const int64_t gy = ceil_div(a_rows, 32);
  LCRW_REQUIRE(gy < 65536, "lcrw_table_transpose: query vocabulary too large for one launch");
  cudaStream_t st = as_stream(stream);
  if (a_rows % tbl::kChunk) {  // fields of words past a_rows in the last chunk: defined zeros
    const int64_t last = a_rows / tbl::kChunk;
    cudaError_t e = cudaMemsetAsync(static_cast<uint8_t*>(T) + last * v_rows * kTableRowBytes, 0,
                                    (size_t)v_rows * kTableRowBytes, st);
    if (e != cudaSuccess) return cuda_status(e, "cudaMemsetAsync (table tail)");
  }
  ProfScope prof(st, "table_transpose");
  tbl::transpose_kernel<<<dim3((unsigned)ceil_div(v_rows, 32), (unsigned)gy), 256, 0, st>>>(
      Tp, a_norms, a_rows, v_rows, scale, static_cast<uint8_t*>(T));
  LCRW_CHECK_LAUNCH("table_transpose_kernel");
  return LCRW_OK;
}

int lcrw_table_min(const void* T, int64_t a_rows, int64_t v_rows, const int64_t* doc_offsets, int64_t seg_base,
                   int64_t n_docs, const int32_t* doc_cols, const float* scale, float* Z2, int64_t z_panel,
                   const float* a_norms, void* refine_list, uint64_t* refine_count, int64_t refine_cap,
                   void* stream) {
  LCRW_REQUIRE(a_rows >= 0 && v_rows >= 0 && n_docs >= 0, "lcrw_table_min: bad shape");
  if (a_rows == 0 || n_docs == 0) return LCRW_OK;
  LCRW_REQUIRE(T && doc_offsets && doc_cols && Z2 && scale, "lcrw_table_min: null pointer");
  LCRW_REQUIRE(!refine_list || (a_norms && refine_count && refine_cap >= 0),
               "lcrw_table_min: a refine list needs a_norms, its count and capacity");
  LCRW_REQUIRE(z_panel == a_rows * tbl::kPanelDocs && (reinterpret_cast<uintptr_t>(T) & 15) == 0,
               "lcrw_table_min: Z2 must be in 32-doc panels (z_panel = 32 * a_rows), T 16-byte aligned");
  const int64_t panels = ceil_div(n_docs, tbl::kPanelDocs);
  const int64_t blocks = ceil_div(a_rows, tbl::kChunk) * panels;
  LCRW_REQUIRE(blocks < (1ll << 31), "lcrw_table_min: too many (chunk, panel) blocks for one launch");
  cudaStream_t st = as_stream(stream);
  ProfScope prof(st, "table_min");
  tbl::table_min_kernel<<<(unsigned)blocks, 256, 0, st>>>(static_cast<const uint8_t*>(T), v_rows, a_rows, doc_offsets,
                                                          seg_base, n_docs, doc_cols, scale, Z2, z_panel, panels, a_norms,
      RefineSink{static_cast<uint2*>(refine_list), reinterpret_cast<unsigned long long*>(refine_count), refine_cap});
  LCRW_CHECK_LAUNCH("table_min_kernel");
  return LCRW_OK;
}

}  // extern "C"
