// Exact re-evaluation of near entries of Z (kernels.py:72-110 semantics).
//
// The tensor-core Gram expansion |a|^2 + |b|^2 - 2 a.b carries an absolute error
// that scales with the operands' norms (f16 operand rounding, fp32 accumulation of
// terms ~|a||b|), so a distance much smaller than the norms -- near-duplicate words,
// clustered embeddings -- loses relative precision.  Every Z entry whose (scaled)
// distance d satisfies 0 < d < kRefineTau * |a| is recomputed here as the exact
// segment minimum  min_{b in seg} sqrt(sum_k (a_k - b_k)^2)  from the f32 rows
// (direct differences: no cancellation; fixed summation order, so deterministic).
// Entries at or above the threshold keep the Gram value, whose relative error is
// bounded by the ratio |a| / d <= 1 / kRefineTau (DESIGN.md §5 has the budget).
//
// Two sources of work:
//  * scan: every entry of a Z in (1 << z_shift)-segment panels is tested (forward
//    Z1, pairwise, nearest-word distances -- small Z);
//  * list: the reverse pass's producers (table_min, the GEMM-form Phase-1
//    epilogue) append flagged (row, segment) pairs of their Z2 batch while they
//    write it, with the same test on the same (key-rounded) value, so both forms
//    refine the same entries; a list that overflowed its capacity falls back to
//    the scan (decided on the device, no host sync).
#include "common.cuh"

namespace lcrw {
namespace refine {

constexpr int kThreads = 256;

// sqrt(min over the segment's words of |A[a_id] - B[b_id]|^2), warp-cooperative: lanes
// split the m dimensions, xor-reduction, every lane returns the result
__device__ __forceinline__ float exact_segment_min(const float* __restrict__ a, const float* __restrict__ B, int m,
                                                   const int32_t* __restrict__ seg_ids, int64_t t0, int64_t t1,
                                                   int lane) {
  float best = __int_as_float(0x7f800000);
  for (int64_t t = t0; t < t1; ++t) {
    const float* b = B + (int64_t)__ldg(seg_ids + t) * m;
    float acc = 0.f;
    for (int k = lane; k < m; k += 32) {
      const float diff = __ldg(a + k) - __ldg(b + k);
      acc = fmaf(diff, diff, acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    best = fminf(best, acc);
  }
  return sqrtf(best);
}

struct Args {
  float* Z;
  int64_t z_panel;
  int z_shift;
  int64_t a_rows, n_seg;
  const int64_t* seg_offsets;
  int64_t seg_base;
  const int32_t* seg_ids;
  const float* A32;
  const int32_t* a_ids;
  const float* B32;
  int m;
  const float* a_norms;
  const float* scale;
  const uint2* list;
  const uint32_t* count;
  int64_t cap;
};

__device__ __forceinline__ float* z_at(const Args& g, int64_t row, int64_t s) {
  return g.Z + (s >> g.z_shift) * g.z_panel + (row << g.z_shift) + (s & ((1ll << g.z_shift) - 1));
}

__device__ __forceinline__ void fix(const Args& g, int64_t row, int64_t s, int lane) {
  const float* a = g.A32 + (int64_t)__ldg(g.a_ids + row) * g.m;
  const float d = exact_segment_min(a, g.B32, g.m, g.seg_ids, __ldg(g.seg_offsets + s) - g.seg_base,
                                    __ldg(g.seg_offsets + s + 1) - g.seg_base, lane);
  if (lane == 0) *z_at(g, row, s) = d;
}

#ifndef LCRW_REFINE_MINB
#define LCRW_REFINE_MINB 1
#endif
__global__ void __launch_bounds__(kThreads, LCRW_REFINE_MINB) refine_kernel(Args g) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (blockIdx.x * (int64_t)kThreads + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * kThreads) >> 5;
  if (g.list) {
    const uint32_t n = __ldg(g.count);
    if ((int64_t)n <= g.cap) {
      for (int64_t i = warp0; i < n; i += n_warps) {
        const uint2 e = g.list[i];
        fix(g, e.x, e.y, lane);
      }
      return;
    }
  }
  // scan: panels in order; inside a panel the warps take 128-entry steps, four consecutive
  // entries per lane as one float4 (entry i = 128 c + 4 lane + j: row (i >> zs), segment
  // p * zw + (i & (zw - 1))); no division, coalesced 512-byte warp loads, the flagged
  // entries (rare) fixed one at a time by the whole warp
  const float s0 = __ldg(g.scale);
  const float tau2 = kRefineTau * kRefineTau;
  const int64_t zw = 1ll << g.z_shift;
  const int64_t per_panel = g.a_rows << g.z_shift;  // a multiple of 4 (z_shift >= 2)
  const int64_t cpp = (per_panel + 127) >> 7;       // 128-entry steps per panel
  const int64_t n_panels = (g.n_seg + zw - 1) >> g.z_shift;
  constexpr int kSteps = 4;  // 128-entry steps in flight per warp (independent loads)
  for (int64_t p = 0; p < n_panels; ++p) {
    const float* zp = g.Z + p * g.z_panel;
    const int64_t seg_left = g.n_seg - p * zw;  // < zw only in a ragged last panel
    for (int64_t c0 = warp0; c0 < cpp; c0 += kSteps * n_warps) {
      float4 z4[kSteps];
#pragma unroll
      for (int u = 0; u < kSteps; ++u) {
        const int64_t i0 = ((c0 + u * n_warps) << 7) + 4 * lane;
        z4[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (i0 < per_panel) {
          const int64_t sl = i0 & (zw - 1);  // segment of the lane's first entry inside the panel
          if (sl + 4 <= seg_left) {
            z4[u] = __ldg(reinterpret_cast<const float4*>(zp + i0));
          } else {  // entries past the last segment hold no values: not read
            if (sl + 0 < seg_left) z4[u].x = __ldg(zp + i0);
            if (sl + 1 < seg_left) z4[u].y = __ldg(zp + i0 + 1);
            if (sl + 2 < seg_left) z4[u].z = __ldg(zp + i0 + 2);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kSteps; ++u) {
        const int64_t c = c0 + u * n_warps;
        const int64_t i0 = (c << 7) + 4 * lane;
        uint32_t flags = 0;
        if (i0 < per_panel) {
          // the lane's four entries share one row (z_shift >= 2): one norm, one bound
          const float zv[4] = {z4[u].x, z4[u].y, z4[u].z, z4[u].w};
          if (zv[0] > 0.f || zv[1] > 0.f || zv[2] > 0.f || zv[3] > 0.f) {
            const float a_sq = __ldg(g.a_norms + (i0 >> g.z_shift));
            const int64_t s_base = p * zw + (i0 & (zw - 1));
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (s_base + j < g.n_seg && refine_flag(zv[j] * s0, a_sq, tau2)) flags |= 1u << j;
          }
        }
        if (__any_sync(0xffffffffu, flags != 0)) {  // rare: fix the warp's flagged entries one by one
#pragma unroll 1
          for (int j = 0; j < 4; ++j) {
            uint32_t ballot = __ballot_sync(0xffffffffu, (flags >> j) & 1u);
            while (ballot) {
              const int src = __ffs(ballot) - 1;
              ballot &= ballot - 1u;
              const int64_t i = (c << 7) + 4 * src + j;
              fix(g, i >> g.z_shift, p * zw + (i & (zw - 1)), lane);
            }
          }
        }
      }
    }
  }
}

}  // namespace refine
}  // namespace lcrw

using namespace lcrw;

extern "C" {

float lcrw_refine_tau(void) { return kRefineTau; }

int lcrw_refine_near(float* Z, int64_t z_panel, int z_shift, int64_t a_rows, int64_t n_seg,
                     const int64_t* seg_offsets, int64_t seg_base, const int32_t* seg_ids, const float* A32,
                     const int32_t* a_ids, const float* B32, int m, const float* a_norms, const float* scale,
                     const void* list, const uint32_t* count, int64_t cap, void* stream) {
  LCRW_REQUIRE(a_rows >= 0 && n_seg >= 0 && m > 0, "lcrw_refine_near: bad shape");
  if (a_rows == 0 || n_seg == 0) return LCRW_OK;
  LCRW_REQUIRE(Z && seg_offsets && seg_ids && A32 && a_ids && B32 && a_norms && scale,
               "lcrw_refine_near: null pointer");
  LCRW_REQUIRE(z_shift >= 2 && z_shift <= 10 && z_panel >= (a_rows << z_shift) && z_panel % 4 == 0 &&
                   (reinterpret_cast<uintptr_t>(Z) & 15) == 0,
               "lcrw_refine_near: bad Z layout (z_shift in [2, 10], z_panel % 4 == 0, Z 16-byte aligned)");
  LCRW_REQUIRE(!list || (count && cap >= 0), "lcrw_refine_near: a list needs its count and capacity");
  refine::Args g{Z, z_panel, z_shift, a_rows, n_seg, seg_offsets, seg_base, seg_ids, A32, a_ids, B32, m, a_norms,
                 scale, static_cast<const uint2*>(list), count, cap};
  const int64_t entries = ((n_seg + (1ll << z_shift) - 1) >> z_shift) * (a_rows << z_shift);
  const int64_t want = ceil_div(entries, (int64_t)refine::kThreads);
  const int64_t cap_blocks = (int64_t)sm_count() * 16;
  const int blocks = (int)(want < cap_blocks ? (want > 0 ? want : 1) : cap_blocks);
  cudaStream_t st = as_stream(stream);
  ProfScope prof(st, "refine");
  refine::refine_kernel<<<blocks, refine::kThreads, 0, st>>>(g);
  LCRW_CHECK_LAUNCH("refine_kernel");
  return LCRW_OK;
}

}  // extern "C"
