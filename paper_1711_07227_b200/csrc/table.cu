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
namespace tbl {

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
  for (int dd = warp; dd < kPanelDocs; dd += 8) {
    const int64_t d = p * kPanelDocs + dd;
    float4 acc = make_float4(inf, inf, inf, inf);
    if (d < n_docs) {
      const int64_t b = __ldg(doc_offsets + d) - seg_base, e = __ldg(doc_offsets + d + 1) - seg_base;
      for (int64_t j0 = b; j0 < e; j0 += 32) {
        const int n = e - j0 < 32 ? (int)(e - j0) : 32;
        const int mine = lane < n ? __ldg(cols + j0 + lane) : 0;
#pragma unroll 8
        for (int j = 0; j < n; ++j) {
          const int u = __shfl_sync(0xffffffffu, mine, j);
          const float4 x = __ldg(Tc + (int64_t)u * (kChunk / 4));
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
    if (w + 0 < a_rows) zp[(w + 0) * kPanelDocs + lane] = v.x;
    if (w + 1 < a_rows) zp[(w + 1) * kPanelDocs + lane] = v.y;
    if (w + 2 < a_rows) zp[(w + 2) * kPanelDocs + lane] = v.z;
    if (w + 3 < a_rows) zp[(w + 3) * kPanelDocs + lane] = v.w;
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
