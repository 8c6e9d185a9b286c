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
// the exact zeros, transposes it into 128-word chunks [chunk][u][128 w] (one
// 512-byte row per vocabulary word), and then each doc's Z2 column is a
// min over its words' rows: 512-byte gathers from an L2-resident 51 MB chunk
// (V = 100k), L2-bandwidth bound instead of tensor bound.
#include "common.cuh"

namespace lcrw {
namespace p1 {
int launch(const uint16_t* A, const float* a_norms, int64_t a_rows, const uint16_t* B, int64_t b_rows, int m, int kp,
           const int64_t* seg_offsets, int64_t seg_base, int64_t n_seg, const uint32_t* endmask,
           const int32_t* range_seg, int64_t n_ranges, const float* scale, float* Z, int64_t z_panel, int z_shift,
           cudaStream_t stream, const char* tag, const int32_t* b_ids, int64_t b_table_rows, bool z_transposed);
}
namespace tbl {

#ifndef LCRW_TBL_HINTS
#define LCRW_TBL_HINTS 1
#endif

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
__device__ __forceinline__ float4 ld_keep(const float4* ptr, uint64_t pol) {
#if LCRW_TBL_HINTS
  float4 v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "l"(ptr), "l"(pol));
  return v;
#else
  return __ldg(ptr);
#endif
}
__device__ __forceinline__ int ld_stream(const int32_t* ptr, uint64_t pol) {
#if LCRW_TBL_HINTS
  int v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(ptr), "l"(pol));
  return v;
#else
  return __ldg(ptr);
#endif
}
__device__ __forceinline__ void st_stream(float* ptr, float v, uint64_t pol) {
#if LCRW_TBL_HINTS
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(ptr), "f"(v), "l"(pol) : "memory");
#else
  *ptr = v;
#endif
}

constexpr int kChunk = 128;        // query-vocabulary words per table chunk (512-byte rows)
constexpr int kPanelDocs = 32;     // Z2 panel width (lcrw_reverse_panels layout)

// T'[(u >> 7) * zp + (w << 7) + (u & 127)] (lcrw_phase1 layout, z_shift 7, zp = a_rows * 128)
//   -> T[(w >> 7) * v_rows * 128 + (u << 7) + (w & 127)]; padded words (w >= a_rows) get 0.
__global__ void __launch_bounds__(256) transpose_kernel(const float* __restrict__ Tp, int64_t a_rows, int64_t v_rows,
                                                        float* __restrict__ T) {
  __shared__ float t[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t u0 = (int64_t)blockIdx.x * 32, w0 = (int64_t)blockIdx.y * 32;
  const int64_t zp = a_rows * kChunk;
  for (int y = ty; y < 32; y += 8) {  // source rows w0 + y, columns u0 + tx (contiguous in u)
    const int64_t w = w0 + y, u = u0 + tx;
    t[y][tx] = (w < a_rows && u < v_rows) ? Tp[(u >> 7) * zp + (w << 7) + (u & 127)] : 0.f;
  }
  __syncthreads();
  for (int y = ty; y < 32; y += 8) {  // destination rows u0 + y, columns w0 + tx (contiguous in w)
    const int64_t u = u0 + y, w = w0 + tx;
    if (u < v_rows) T[(w >> 7) * v_rows * kChunk + (u << 7) + (w & 127)] = t[tx][y];
  }
}

// Exact zeros (kernels.py:91-92, as lcrw_zero_identical): T[w, u] = 0 for every query-
// vocabulary row w whose E row is bitwise identical to E row u (class chain of canon[u]).
__global__ void table_zeros_kernel(const int32_t* __restrict__ canon, const int32_t* __restrict__ next,
                                   const int32_t* __restrict__ remap, int64_t v_rows, float* __restrict__ T) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < v_rows;
       u += (int64_t)gridDim.x * blockDim.x) {
    for (int32_t g = canon[u]; g >= 0; g = next[g]) {
      const int32_t r = remap[g];
      if (r >= 0) T[((int64_t)r >> 7) * v_rows * kChunk + (u << 7) + (r & 127)] = 0.f;
    }
  }
}

// One CTA per (chunk c, 32-doc panel p), panels fastest so the CTAs in flight
// share one L2-resident chunk.  Warp j takes docs j, j+8, j+16, j+24; lane l owns
// words 4l..4l+3 of the chunk (one float4 of each 512-byte row).  The 32 x 128
// result is staged in smem (float4 XOR swizzle: conflict-free both ways) and
// written as 128 coalesced 128-byte Z2 rows: Z2[p * z_panel + w * 32 + doc].
__global__ void __launch_bounds__(256) table_min_kernel(const float4* __restrict__ T, int64_t v_rows, int64_t a_rows,
                                                        const int64_t* __restrict__ doc_offsets, int64_t seg_base,
                                                        int64_t n_docs, const int32_t* __restrict__ cols,
                                                        float* __restrict__ Z2, int64_t z_panel, int64_t panels) {
  __shared__ float4 tile[kPanelDocs][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t c = blockIdx.x / panels, p = blockIdx.x - c * panels;
  const float4* Tc = T + c * v_rows * (kChunk / 4) + lane;
  const float inf = __int_as_float(0x7f800000);
  const uint64_t keep = l2_policy_last(), stream = l2_policy_first();
  for (int dd = warp; dd < kPanelDocs; dd += 8) {
    const int64_t d = p * kPanelDocs + dd;
    float4 acc = make_float4(inf, inf, inf, inf);
    if (d < n_docs) {
      const int64_t b = __ldg(doc_offsets + d) - seg_base, e = __ldg(doc_offsets + d + 1) - seg_base;
      for (int64_t j0 = b; j0 < e; j0 += 32) {
        const int n = e - j0 < 32 ? (int)(e - j0) : 32;
        const int mine = lane < n ? ld_stream(cols + j0 + lane, stream) : 0;
#pragma unroll 8
        for (int j = 0; j < n; ++j) {
          const int u = __shfl_sync(0xffffffffu, mine, j);
          const float4 x = ld_keep(Tc + (int64_t)u * (kChunk / 4), keep);
          acc.x = fminf(acc.x, x.x);
          acc.y = fminf(acc.y, x.y);
          acc.z = fminf(acc.z, x.z);
          acc.w = fminf(acc.w, x.w);
        }
      }
    }
    tile[dd][lane ^ (dd & 7)] = acc;
  }
  __syncthreads();
  float* zp = Z2 + p * z_panel;
  for (int q = warp; q < 32; q += 8) {  // lane = doc; words 4q..4q+3
    const float4 v = tile[lane][q ^ (lane & 7)];
    const int64_t w = c * kChunk + 4 * q;
    if (w + 0 < a_rows) st_stream(zp + (w + 0) * kPanelDocs + lane, v.x, stream);
    if (w + 1 < a_rows) st_stream(zp + (w + 1) * kPanelDocs + lane, v.y, stream);
    if (w + 2 < a_rows) st_stream(zp + (w + 2) * kPanelDocs + lane, v.z, stream);
    if (w + 3 < a_rows) st_stream(zp + (w + 3) * kPanelDocs + lane, v.w, stream);
  }
}

}  // namespace tbl
}  // namespace lcrw

using namespace lcrw;

extern "C" {

int lcrw_table_chunk(void) { return tbl::kChunk; }

int64_t lcrw_table_floats(int64_t a_rows, int64_t v_rows) {
  return ceil_div(a_rows, tbl::kChunk) * v_rows * tbl::kChunk;
}

int lcrw_distance_table(const uint16_t* A, const float* a_norms, int64_t a_rows, const uint16_t* EhB, int64_t v_rows,
                        int m, int kp, const int64_t* seg_offsets, const uint32_t* endmask, const int32_t* range_seg,
                        int64_t n_ranges, const float* scale, const int32_t* canon, const int32_t* next,
                        const int32_t* remap, float* T, void* stream) {
  LCRW_REQUIRE(a_rows >= 0 && v_rows >= 0, "lcrw_distance_table: bad shape");
  if (a_rows == 0 || v_rows == 0) return LCRW_OK;
  LCRW_REQUIRE(canon && next && remap && T, "lcrw_distance_table: null pointer");
  cudaStream_t st = as_stream(stream);
  int status = p1::launch(A, a_norms, a_rows, EhB, v_rows, m, kp, seg_offsets, 0, v_rows, endmask, range_seg,
                          n_ranges, scale, T, v_rows * tbl::kChunk, 7, st, "table_build", nullptr, 0, true);
  if (status) return status;
  const int64_t blocks = ceil_div(v_rows, 256);
  tbl::table_zeros_kernel<<<(unsigned)(blocks < 4096 ? blocks : 4096), 256, 0, st>>>(canon, next, remap, v_rows, T);
  LCRW_CHECK_LAUNCH("table_zeros_kernel");
  return LCRW_OK;
}

int lcrw_table_transpose(const float* Tp, int64_t a_rows, int64_t v_rows, float* T, void* stream) {
  LCRW_REQUIRE(a_rows >= 0 && v_rows >= 0, "lcrw_table_transpose: bad shape");
  if (a_rows == 0 || v_rows == 0) return LCRW_OK;
  LCRW_REQUIRE(Tp && T, "lcrw_table_transpose: null pointer");
  const int64_t gy = ceil_div(a_rows, tbl::kChunk) * (tbl::kChunk / 32);
  LCRW_REQUIRE(gy < 65536, "lcrw_table_transpose: query vocabulary too large for one launch");
  cudaStream_t st = as_stream(stream);
  ProfScope prof(st, "table_transpose");
  tbl::transpose_kernel<<<dim3((unsigned)ceil_div(v_rows, 32), (unsigned)gy), 256, 0, st>>>(Tp, a_rows, v_rows, T);
  LCRW_CHECK_LAUNCH("table_transpose_kernel");
  return LCRW_OK;
}

int lcrw_table_min(const float* T, int64_t a_rows, int64_t v_rows, const int64_t* doc_offsets, int64_t seg_base,
                   int64_t n_docs, const int32_t* doc_cols, float* Z2, int64_t z_panel, void* stream) {
  LCRW_REQUIRE(a_rows >= 0 && v_rows >= 0 && n_docs >= 0, "lcrw_table_min: bad shape");
  if (a_rows == 0 || n_docs == 0) return LCRW_OK;
  LCRW_REQUIRE(T && doc_offsets && doc_cols && Z2, "lcrw_table_min: null pointer");
  LCRW_REQUIRE(z_panel == a_rows * tbl::kPanelDocs && (reinterpret_cast<uintptr_t>(T) & 15) == 0,
               "lcrw_table_min: Z2 must be in 32-doc panels (z_panel = 32 * a_rows), T 16-byte aligned");
  const int64_t panels = ceil_div(n_docs, tbl::kPanelDocs);
  const int64_t blocks = ceil_div(a_rows, tbl::kChunk) * panels;
  LCRW_REQUIRE(blocks < (1ll << 31), "lcrw_table_min: too many (chunk, panel) blocks for one launch");
  cudaStream_t st = as_stream(stream);
  ProfScope prof(st, "table_min");
  tbl::table_min_kernel<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<const float4*>(T), v_rows, a_rows,
                                                          doc_offsets, seg_base, n_docs, doc_cols, Z2, z_panel,
                                                          panels);
  LCRW_CHECK_LAUNCH("table_min_kernel");
  return LCRW_OK;
}

}  // extern "C"
