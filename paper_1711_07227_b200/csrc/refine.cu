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
// and three modes:
//  * fix: flagged entries are recomputed here;
//  * mark: flagged entries are set to kZMarked and counted (no arithmetic) so that
//    lcrw_near_scatter can lower them to their exact minimum from the near-pair lists;
//  * finalize: marked entries (the producer's or mark's) get their mark bit cleared, or,
//    when no near pair reached them (still kZMarked), the exact segment minimum.
// The three give bitwise the same Z (a near-pair minimum is certified equal
// to the exact segment minimum).
#include "common.cuh"

namespace lcrw {
namespace refine {

constexpr int kThreads = 256;

// sqrt(min over the segment's words of |A[a_id] - B[b_id]|^2); every lane returns it
__device__ __forceinline__ float exact_segment_min(const float* __restrict__ a, const float* __restrict__ B, int m,
                                                   const int32_t* __restrict__ seg_ids, int64_t t0, int64_t t1,
                                                   int lane) {
  float best = __int_as_float(0x7f800000);
  for (int64_t t = t0; t < t1; ++t) best = fminf(best, exact_sq(a, B + (int64_t)__ldg(seg_ids + t) * m, m, lane));
  return sqrtf(best);
}

enum Mode { kFix = 0, kMark = 1, kFinalize = 2, kKeyed = 4 };

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
  unsigned long long* count;
  int64_t cap;
  int mode;
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
#define LCRW_REFINE_MINB 3  // 3 CTAs (24 warps) per SM: <= 85 registers, no spills
#endif
// one instantiation per mode (kMode = g.mode): the scan loop carries only its mode's work
// (c4 scan 174 -> 153 ms per step, c5 11.4 -> 9.6 ms; 4 CTAs/SM at 64 registers or an
// out-of-line fix() measured slower)
template <int kMode>
__global__ void __launch_bounds__(kThreads, LCRW_REFINE_MINB) refine_kernel(Args g) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (blockIdx.x * (int64_t)kThreads + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * kThreads) >> 5;
  constexpr bool finalize = (kMode & 3) == kFinalize, mark = (kMode & 3) == kMark;
  constexpr bool keyed = (kMode & kKeyed) != 0;  // Z holds 16-bit key values: saturated ones are flagged too
  if (finalize && __ldg(g.count) == 0) return;  // nothing was marked
  if (g.list && !mark) {
    const unsigned long long n = __ldg(g.count);
    if (n <= (unsigned long long)g.cap) {
      for (int64_t i = warp0; i < (int64_t)n; i += n_warps) {
        const uint2 e = g.list[i];
        if (finalize) {
          uint32_t* z = reinterpret_cast<uint32_t*>(z_at(g, e.x, e.y));
          const uint32_t bits = *z;  // (the listed entries are distinct: one warp each)
          if (bits == kZMarked) fix(g, e.x, e.y, lane);
          else if (lane == 0 && (bits & kZMarkBit)) *z = bits & ~kZMarkBit;
        } else {
          fix(g, e.x, e.y, lane);
        }
      }
      return;
    }
  }
  // scan: the (panel, 128-entry step) pairs in panel order, warp w taking pairs w, w + n_warps,
  // ..., kSteps at a time; four consecutive entries per lane as one float4 (entry i = 128 c
  // + 4 lane + j of panel p: row (i >> zs), segment p * zw + (i & (zw - 1))); coalesced
  // 512-byte warp loads, the flagged entries (rare) fixed one at a time by the whole warp
  const float s0 = __ldg(g.scale);
  const float tau2 = kRefineTau * kRefineTau;
  const int64_t zw = 1ll << g.z_shift;
  const int64_t per_panel = g.a_rows << g.z_shift;  // a multiple of 4 (z_shift >= 2)
  const int64_t cpp = (per_panel + 127) >> 7;       // 128-entry steps per panel
  const int64_t n_panels = (g.n_seg + zw - 1) >> g.z_shift;
  const int64_t total = n_panels * cpp;
  constexpr int kSteps = 4;  // steps in flight per warp (independent loads)
  // (panel, step) of the warp's next pair, advanced by n_warps pairs without division
  // (32-bit: panels and steps per panel < 2^31 -- lcrw_refine_near checks)
  const int32_t dp = (int32_t)(n_warps / cpp), dc = (int32_t)(n_warps - (int64_t)dp * cpp);
  int32_t pn = (int32_t)(warp0 / cpp), cn = (int32_t)(warp0 - (int64_t)pn * cpp);
  unsigned long long marked = 0;
  for (int64_t st0 = warp0; st0 < total; st0 += kSteps * n_warps) {
    int32_t pu[kSteps], cu[kSteps];
#pragma unroll
    for (int u = 0; u < kSteps; ++u) {
      pu[u] = pn;
      cu[u] = cn;
      cn += dc;
      pn += dp;
      if (cn >= cpp) {
        cn -= cpp;
        ++pn;
      }
    }
    {
      float4 z4[kSteps];
      float a_sq4[kSteps];  // the rows' norms, loaded with the entries (not after a test on them)
#pragma unroll
      for (int u = 0; u < kSteps; ++u) {
        const int64_t i0 = ((int64_t)cu[u] << 7) + 4 * lane;
        const float* zp = g.Z + pu[u] * g.z_panel;
        const int64_t seg_left = g.n_seg - (int64_t)pu[u] * zw;  // < zw only in a ragged last panel
        z4[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        a_sq4[u] = 0.f;
        if (pu[u] < n_panels && i0 < per_panel) {
          if (!finalize) a_sq4[u] = __ldg(g.a_norms + (i0 >> g.z_shift));
          const int64_t sl = i0 & (zw - 1);  // segment of the lane's first entry inside the panel
          if (sl + 4 <= seg_left) {
            z4[u] = *reinterpret_cast<const float4*>(zp + i0);
          } else {  // entries past the last segment hold no values: not read
            if (sl + 0 < seg_left) z4[u].x = zp[i0];
            if (sl + 1 < seg_left) z4[u].y = zp[i0 + 1];
            if (sl + 2 < seg_left) z4[u].z = zp[i0 + 2];
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kSteps; ++u) {
        const int64_t p = pu[u], c = cu[u];
        float* zp = g.Z + p * g.z_panel;
        const int64_t seg_left = g.n_seg - p * zw;
        const int64_t i0 = (c << 7) + 4 * lane;
        uint32_t flags = 0;
        const float zv[4] = {z4[u].x, z4[u].y, z4[u].z, z4[u].w};
        if (p < n_panels && i0 < per_panel) {
          if (finalize) {  // marked entries (padding past the last segment reads as 0)
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (__float_as_uint(zv[j]) & kZMarkBit) flags |= 1u << j;
          } else if (zv[0] > 0.f || zv[1] > 0.f || zv[2] > 0.f || zv[3] > 0.f) {
            // the lane's four entries share one row (z_shift >= 2): one norm, one bound
            const float a_sq = a_sq4[u];
            const float sat = keyed ? key16_sat(key16_base(a_sq)) : __int_as_float(0x7f800000);
            const int64_t s_base = p * zw + (i0 & (zw - 1));
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (s_base + j < g.n_seg && (refine_flag(zv[j] * s0, a_sq, tau2) || zv[j] * s0 >= sat))
                flags |= 1u << j;
          }
        }
        if (mark || finalize) {
          // lane-local: mark the flagged entries (mark), or clear the marks of the entries a
          // near pair reached (finalize); one 16-byte store when the four are in bounds
          uint32_t w[4], changed = 0;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            w[j] = __float_as_uint(zv[j]);
            if ((flags >> j) & 1u) {
              if (mark) {
                w[j] = kZMarked;
                changed |= 1u << j;
              } else if (w[j] != kZMarked) {
                w[j] &= ~kZMarkBit;
                changed |= 1u << j;
                flags &= ~(1u << j);
              }
            }
          }
          if (changed) {
            uint32_t* zw32 = reinterpret_cast<uint32_t*>(zp) + i0;
            if ((i0 & (zw - 1)) + 4 <= seg_left) {
              *reinterpret_cast<uint4*>(zw32) = make_uint4(w[0], w[1], w[2], w[3]);
            } else {
#pragma unroll
              for (int j = 0; j < 4; ++j)
                if ((changed >> j) & 1u) zw32[j] = w[j];
            }
          }
          if (mark) {
            marked += __popc(flags);
            continue;
          }
          __syncwarp();  // the stores above before any lane's fix of the same words
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
  if (mark) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) marked += __shfl_xor_sync(0xffffffffu, marked, o);
    if (lane == 0 && marked) atomicAdd(g.count, marked);
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
                     const void* list, uint64_t* count, int64_t cap, int mode, void* stream) {
  LCRW_REQUIRE(a_rows >= 0 && n_seg >= 0 && m > 0, "lcrw_refine_near: bad shape");
  if (a_rows == 0 || n_seg == 0) return LCRW_OK;
  LCRW_REQUIRE(Z && seg_offsets && seg_ids && A32 && a_ids && B32 && a_norms && scale,
               "lcrw_refine_near: null pointer");
  LCRW_REQUIRE(z_shift >= 2 && z_shift <= 10 && z_panel >= (a_rows << z_shift) && z_panel % 4 == 0 &&
                   (reinterpret_cast<uintptr_t>(Z) & 15) == 0,
               "lcrw_refine_near: bad Z layout (z_shift in [2, 10], z_panel % 4 == 0, Z 16-byte aligned)");
  LCRW_REQUIRE(ceil_div(n_seg, 1ll << z_shift) < (1ll << 31) && ceil_div(a_rows << z_shift, 128) < (1ll << 31),
               "lcrw_refine_near: Z too large");
  LCRW_REQUIRE((mode & ~4) >= 0 && (mode & ~4) <= 2,
               "lcrw_refine_near: mode is 0 (fix), 1 (mark) or 2 (finalize), | 4 for keyed values");
  LCRW_REQUIRE(!list || (count && cap >= 0), "lcrw_refine_near: a list needs its count and capacity");
  LCRW_REQUIRE((mode & 3) == 0 || count, "lcrw_refine_near: mark and finalize need the count");
  refine::Args g{Z, z_panel, z_shift, a_rows, n_seg, seg_offsets, seg_base, seg_ids, A32, a_ids, B32, m, a_norms,
                 scale, static_cast<const uint2*>(list), reinterpret_cast<unsigned long long*>(count), cap, mode};
  // one warp per 128-entry step (scan) or list entry, at most one resident wave of CTAs
  const int64_t steps = ((n_seg + (1ll << z_shift) - 1) >> z_shift) * ceil_div(a_rows << z_shift, 128);
  const int64_t want = ceil_div(steps, (int64_t)(refine::kThreads / 32));
  void (*kern)(refine::Args) = nullptr;
  switch (mode) {
    case 0: kern = refine::refine_kernel<0>; break;
    case 1: kern = refine::refine_kernel<1>; break;
    case 2: kern = refine::refine_kernel<2>; break;
    case 4: kern = refine::refine_kernel<4>; break;
    case 5: kern = refine::refine_kernel<5>; break;
    default: kern = refine::refine_kernel<6>; break;
  }
  static int per_sm[7] = {0, 0, 0, 0, 0, 0, 0};
  if (!per_sm[mode]) {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, refine::kThreads, 0) != cudaSuccess || n < 1) n = 1;
    per_sm[mode] = n;
  }
  const int64_t cap_blocks = (int64_t)sm_count() * per_sm[mode];
  const int blocks = (int)(want < cap_blocks ? (want > 0 ? want : 1) : cap_blocks);
  cudaStream_t st = as_stream(stream);
  ProfScope prof(st, "refine");
  kern<<<blocks, refine::kThreads, 0, st>>>(g);
  LCRW_CHECK_LAUNCH("refine_kernel");
  return LCRW_OK;
}

}  // extern "C"
