// Phase 2 of LC-RWMD (kernels.py:174-198 spmm, distances.py:203) and the
// reverse direction's Phase 2 with the fused symmetric combine
// (distances.py:263-264); the per-query top-k over the result is in topk.cu.
//
// Both kernels read Z in the 8-segment panel layout written by Phase 1
// (Z[(s>>3)*z_panel + row*8 + (s&7)]) so that a warp's lanes touch whole
// 32-byte sectors.  Products and sums are fp64 in ascending nonzero order,
// rounded once to f32 -- the reference's arithmetic (kernels.py:188-190), so
// given the same Z the result is bitwise identical.
#include "common.cuh"

namespace lcrw {
namespace p2 {

constexpr int kWarps = 8;
constexpr int kSegPerBlock = 128;   // spmm: 32 lanes x 4 segments

// ---------------------------------------------------------------------------
// CSR x panelled Z: one warp per CSR row, 4 consecutive segments per lane.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kWarps * 32)
    spmm_kernel(const int64_t* __restrict__ offs, const int32_t* __restrict__ cols, const float* __restrict__ vals,
                int64_t n_rows, const float* __restrict__ Z, int64_t z_panel, int64_t z_block_rows,
                int64_t z_block_stride, int64_t n_seg, float* __restrict__ out, int64_t ld_row, int64_t ld_panel) {
  const int lane = threadIdx.x & 31;
  const int64_t q0 = (int64_t)blockIdx.y * kSegPerBlock + lane * 4;
  const bool active = q0 < n_seg;
  const float* zq = Z + (q0 >> 3) * z_panel + (q0 & 7);
  const uint32_t zbr = (uint32_t)min(z_block_rows, (int64_t)0xFFFFFFFF);
  for (int64_t i = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); i < n_rows; i += (int64_t)gridDim.x * kWarps) {
    const int64_t lo = offs[i], hi = offs[i + 1];
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    for (int64_t base = lo; base < hi; base += 32) {
      const int cnt = (int)min((int64_t)32, hi - base);
      const uint32_t my_c = lane < cnt ? (uint32_t)__ldg(cols + base + lane) : 0u;
      const float my_x = lane < cnt ? __ldg(vals + base + lane) : 0.f;
      // vocabulary-sliced Z (multi-GPU all-gather): row w lives in block w / z_block_rows
      const uint32_t blk = my_c / zbr;
      const int64_t my_off = (int64_t)blk * z_block_stride + (int64_t)(my_c - blk * zbr) * 8;
      for (int t = 0; t < cnt; ++t) {
        const int64_t zoff = __shfl_sync(0xffffffffu, my_off, t);
        const double x = (double)__shfl_sync(0xffffffffu, my_x, t);
        if (active) {
          const float4 z = __ldg(reinterpret_cast<const float4*>(zq + zoff));
          a0 = fma(x, (double)z.x, a0);
          a1 = fma(x, (double)z.y, a1);
          a2 = fma(x, (double)z.z, a2);
          a3 = fma(x, (double)z.w, a3);
        }
      }
    }
    if (active) {
      const double a[4] = {a0, a1, a2, a3};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t q = q0 + e;
        if (q < n_seg) out[i * ld_row + (q >> 3) * ld_panel + (q & 7)] = (float)a[e];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Reverse direction, panel-streaming form.  One CTA per (32-doc Z2 panel,
// group of <= 1024 queries): the panel's word rows are streamed through shared
// memory in 256-row tiles (cp.async, sequential 32 KB reads -- each Z2 byte is
// read from HBM once), and a word-major list of the query nonzeros scatters
// x * Z2[w, 32 docs] into per-query fp32 accumulators in shared memory.  Each
// query is owned by one warp (q % 16), so accumulation order is fixed (tile,
// then row): results are deterministic.  The symmetric combine max(D1, D2) is
// written query-major (128-byte rows) for the final per-query top-k.
// ---------------------------------------------------------------------------
constexpr int kRpWarps = 16;   // consumer warps (+1 producer warp)
constexpr int kRpTile = 128;   // Z2 rows per staged tile (16 KB)
constexpr int kRpStages = 4;
constexpr int kRpGroup = 1024; // queries per CTA

__global__ void __launch_bounds__((kRpWarps + 1) * 32, 1)
    reverse_panels_kernel(const float* __restrict__ Z2, int64_t z_panel, int64_t a_rows, int64_t n_docs,
                          int64_t doc_base, const uint32_t* __restrict__ e_pack, const float* __restrict__ e_x,
                          const int32_t* __restrict__ e_off, int n_tiles, int64_t n_q, const float* __restrict__ D1,
                          int64_t d1_ld_panel, float* __restrict__ D, int64_t ld_q, int64_t ld_doc) {
  extern __shared__ __align__(16) float rp_smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t p = blockIdx.x;
  const int g = blockIdx.y;
  const int64_t q0 = (int64_t)g * kRpGroup;
  const int nq = (int)min((int64_t)kRpGroup, n_q - q0);
  float* acc = rp_smem;                                              // [kRpGroup][32]
  float* tiles = rp_smem + (size_t)kRpGroup * 32;                    // [kRpStages][kRpTile][32]
  uint64_t* full = reinterpret_cast<uint64_t*>(tiles + kRpStages * kRpTile * 32);
  uint64_t* empty = full + kRpStages;
  int32_t* offs = reinterpret_cast<int32_t*>(empty + kRpStages);    // [n_tiles * W + 1]
  const int32_t* goff = e_off + (int64_t)g * n_tiles * kRpWarps;
  for (int i = threadIdx.x; i <= n_tiles * kRpWarps; i += blockDim.x) offs[i] = __ldg(goff + i);
  for (int i = threadIdx.x; i < nq * 32; i += blockDim.x) acc[i] = 0.f;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kRpStages; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, kRpWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const float* zp = Z2 + p * z_panel;

  if (warp == kRpWarps) {
    // ---- producer: stream the panel's rows, kRpStages tiles ahead ----
    if (lane == 0) {
      for (int t = 0; t < n_tiles; ++t) {
        const int st = t % kRpStages;
        mbar_wait(empty + st, ((t / kRpStages) & 1) ^ 1);
        const int64_t r0 = (int64_t)t * kRpTile;
        const uint32_t bytes = (uint32_t)min((int64_t)kRpTile, a_rows - r0) * 128u;
        mbar_expect_tx(full + st, bytes);
        bulk_load(tiles + st * kRpTile * 32, zp + r0 * 32, bytes, full + st);
      }
    }
  } else {
    // ---- consumers: scatter this warp's query nonzeros of each tile ----
    int e0 = offs[warp], e1 = offs[warp + 1];
    uint32_t pre_p = lane < e1 - e0 ? __ldg(e_pack + e0 + lane) : 0u;
    float pre_x = lane < e1 - e0 ? __ldg(e_x + e0 + lane) : 0.f;
    for (int t = 0; t < n_tiles; ++t) {
      const int st = t % kRpStages;
      // next tile's entry window and first 32 entries (latency hidden behind this tile)
      const int ne0 = t + 1 < n_tiles ? offs[(t + 1) * kRpWarps + warp] : 0;
      const int ne1 = t + 1 < n_tiles ? offs[(t + 1) * kRpWarps + warp + 1] : 0;
      const uint32_t nxt_p = lane < ne1 - ne0 ? __ldg(e_pack + ne0 + lane) : 0u;
      const float nxt_x = lane < ne1 - ne0 ? __ldg(e_x + ne0 + lane) : 0.f;
      mbar_wait(full + st, (t / kRpStages) & 1);
      const float* tile = tiles + st * kRpTile * 32;
      uint32_t cur_p = pre_p;
      float cur_x = pre_x;
      for (int eb = e0; eb < e1; eb += 32) {
        if (eb != e0) {  // rare: more than 32 entries for this (tile, warp)
          cur_p = lane < e1 - eb ? __ldg(e_pack + eb + lane) : 0u;
          cur_x = lane < e1 - eb ? __ldg(e_x + eb + lane) : 0.f;
        }
        const int cnt = min(32, e1 - eb);
        for (int i = 0; i < cnt; ++i) {
          const uint32_t pk = __shfl_sync(0xffffffffu, cur_p, i);
          const float x = __shfl_sync(0xffffffffu, cur_x, i);
          float* a = acc + (pk & 0xFFFFu) * 32 + lane;
          *a = fmaf(x, tile[(pk >> 16) * 32 + lane], *a);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + st);
      e0 = ne0;
      e1 = ne1;
      pre_p = nxt_p;
      pre_x = nxt_x;
    }
  }
  __syncthreads();

  // symmetric combine with D1 (8-query panels: D1[(q >> 3) * ld_panel + j * 8 + (q & 7)])
  const int64_t j = p * 32 + lane;
  const bool valid = j < n_docs;
  const int64_t jg = doc_base + j;
  for (int qp = warp; qp * 8 < nq; qp += kRpWarps + 1) {
    const int64_t qg = q0 + qp * 8;
    float d1v[8];
    if (valid) {
      const float4* src = reinterpret_cast<const float4*>(D1 + (qg >> 3) * d1_ld_panel + jg * 8);
      const float4 a = __ldg(src), b = __ldg(src + 1);
      d1v[0] = a.x; d1v[1] = a.y; d1v[2] = a.z; d1v[3] = a.w;
      d1v[4] = b.x; d1v[5] = b.y; d1v[6] = b.z; d1v[7] = b.w;
    }
#pragma unroll
    for (int qq = 0; qq < 8; ++qq) {
      const int ql = qp * 8 + qq;
      if (valid && ql < nq) D[(qg + qq) * ld_q + jg * ld_doc] = fmaxf(d1v[qq], acc[ql * 32 + lane]);
    }
  }
}


}  // namespace p2
}  // namespace lcrw

using namespace lcrw;
using namespace lcrw::p2;

extern "C" {

int lcrw_spmm(const int64_t* offs, const int32_t* cols, const float* vals, int64_t n_rows, const float* Z,
              int64_t z_panel, int64_t z_block_rows, int64_t z_block_stride, int64_t n_seg, float* out,
              int64_t ld_row, int64_t ld_panel, void* stream) {
  LCRW_REQUIRE(n_rows >= 0 && n_seg >= 0, "lcrw_spmm: bad shape");
  if (n_rows == 0 || n_seg == 0) return LCRW_OK;
  LCRW_REQUIRE(offs && cols && vals && Z && out, "lcrw_spmm: null pointer");
  LCRW_REQUIRE(z_panel % 8 == 0 && z_block_stride % 8 == 0 && (reinterpret_cast<uintptr_t>(Z) & 15) == 0,
               "lcrw_spmm: Z must be 16-byte aligned with z_panel, z_block_stride % 8 == 0");
  if (z_block_rows <= 0) z_block_rows = INT64_MAX;
  const int64_t gy = ceil_div(n_seg, kSegPerBlock);
  LCRW_REQUIRE(gy < 65536, "lcrw_spmm: too many segments for one launch");
  int64_t gx = ceil_div(n_rows, kWarps);
  const int64_t cap = (int64_t)sm_count() * 64;
  if (gx > cap) gx = cap;
  ProfScope prof(as_stream(stream), "spmm");
  spmm_kernel<<<dim3((unsigned)gx, (unsigned)gy), kWarps * 32, 0, as_stream(stream)>>>(
      offs, cols, vals, n_rows, Z, z_panel, z_block_rows, z_block_stride, n_seg, out, ld_row, ld_panel);
  LCRW_CHECK_LAUNCH("spmm_kernel");
  return LCRW_OK;
}


int lcrw_reverse_panels_tile_rows(void) { return kRpTile; }
int lcrw_reverse_panels_group(void) { return kRpGroup; }
int lcrw_reverse_panels_warps(void) { return kRpWarps; }

int lcrw_reverse_panels(const float* Z2, int64_t z_panel, int64_t a_rows, int64_t n_docs, int64_t doc_base,
                        const uint32_t* e_pack, const float* e_x, const int32_t* e_off, int64_t n_q,
                        const float* D1, int64_t d1_ld_panel, float* D, int64_t ld_q, int64_t ld_doc,
                        void* stream) {
  LCRW_REQUIRE(n_q >= 0 && n_docs >= 0 && a_rows >= 0, "lcrw_reverse_panels: bad shape");
  if (n_q == 0 || n_docs == 0) return LCRW_OK;
  LCRW_REQUIRE(Z2 && e_pack && e_x && e_off && D1 && D, "lcrw_reverse_panels: null pointer");
  LCRW_REQUIRE(z_panel == a_rows * 32 && (reinterpret_cast<uintptr_t>(Z2) & 15) == 0,
               "lcrw_reverse_panels: Z2 must be 16-byte aligned 32-doc panels (z_panel = 32 * a_rows)");
  const int n_tiles = (int)ceil_div(a_rows, kRpTile);
  const int64_t panels = ceil_div(n_docs, 32);
  const int64_t groups = ceil_div(n_q, kRpGroup);
  LCRW_REQUIRE(panels < (1ll << 31) && groups < 65536, "lcrw_reverse_panels: grid too large");
  const int fixed = (kRpGroup * 32 + kRpStages * kRpTile * 32) * 4 + 2 * kRpStages * 8;
  const int smem = fixed + (n_tiles * kRpWarps + 1) * 4;
  const int smem_max = 227 * 1024;
  if (smem > smem_max) {
    set_error("lcrw_reverse_panels: query vocabulary of %lld rows needs %d B of shared memory", (long long)a_rows, smem);
    return LCRW_ERR_UNSUPPORTED;
  }
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(reverse_panels_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max);
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(reverse_panels_kernel)");
    attr = true;
  }
  cudaStream_t st = as_stream(stream);
  ProfScope prof(st, "reverse_panels");
  reverse_panels_kernel<<<dim3((unsigned)panels, (unsigned)groups), (kRpWarps + 1) * 32, smem, st>>>(
      Z2, z_panel, a_rows, n_docs, doc_base, e_pack, e_x, e_off, n_tiles, n_q, D1, d1_ld_panel, D, ld_q, ld_doc);
  LCRW_CHECK_LAUNCH("reverse_panels_kernel");
  return LCRW_OK;
}

}  // extern "C"
