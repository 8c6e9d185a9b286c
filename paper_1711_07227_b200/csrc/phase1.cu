// Phase 1 of LC-RWMD on sm_100a (distances.py:147-178, kernels.py:72-110).
//
//   Z[s, r] = min_{t in segment s} sqrt(max(0, |A_r|^2 + |B_t|^2 - 2 A_r . B_t))
//
// A = vocabulary rows (resident side, restricted), B = stacked query-side word
// rows, segments = query histograms.  The dot products run on the 5th-gen
// tensor cores (tcgen05.mma kind::f16, fp32 accumulation in TMEM) fed by TMA;
// the Gram expansion and the segmented row-min are fused into the epilogue so
// the |A| x |B| distance matrix never exists outside TMEM.
//
// CTA pairs (cluster of 2, tcgen05 cta_group::2): one pair computes 256 A rows
// x 256 B rows per tile.  Each CTA keeps ITS 128 A rows (all K blocks) resident
// in shared memory for a whole work unit and streams ITS HALF (128 rows) of
// every B tile through an 8-stage TMA ring; the leader CTA issues the pair MMA
// (M = 256, N = 256, K = 16), whose operands come from both CTAs' smem, and the
// fp32 accumulator rows land in each CTA's own TMEM (2 x 256 columns, double
// buffered).  Splitting B across the pair halves per-SM operand traffic (smem
// reads and L2->SM TMA bytes) relative to a single-CTA M = 128 tile and doubles
// the MMA time each staged byte covers.
//
// Work unit = (pair of 128-row m-tiles, column range of ~range_cols B rows
// bounded by segment boundaries).  Segments may straddle N tiles: the running
// minimum is carried in registers across the tiles of a unit, and ranges never
// cut a segment, so every Z entry is written exactly once (no atomics, no
// initialisation pass).
//
// Warp roles (352 threads per CTA): w0..w7 epilogue (TMEM lane quarter = warp % 4,
// column half = warp / 4, one A row per thread), w8 TMA producer, w9 MMA issuer
// (leader CTA only), w10 TMEM allocator.
#include <cstdio>

#include "common.cuh"

#ifndef LCRW_EPI_MODE
#define LCRW_EPI_MODE 0  // experiment switch: 1 = skip segment minima, 2 = also skip TMEM loads
#endif

namespace lcrw {
namespace p1 {

constexpr int BM = 128;                       // A rows per CTA (TMEM lanes); the pair covers 256
constexpr int BN = 256;                       // B rows per pair tile (MMA N); 128 staged per CTA
constexpr int BN_HALF = BN / 2;
constexpr int BK = 64;                        // f16 elements per K block (128 B rows)
constexpr int A_KB_BYTES = BM * BK * 2;       // 16 KB
constexpr int B_STAGE_BYTES = BN_HALF * BK * 2;  // 16 KB per CTA
constexpr int kEpiWarps = 8;                  // two per TMEM lane quarter: each owns one 128-column half
// Warp roles.  The schedulers favour higher warp ids, so the single-lane TMA and
// MMA issuers sit above the epilogue warps and are never starved by them.
constexpr int kProducerWarp = kEpiWarps;      // 8
constexpr int kMmaWarp = kEpiWarps + 1;       // 9
constexpr int kAllocWarp = kEpiWarps + 2;     // 10
constexpr int kThreads = 32 * (kEpiWarps + 3);
constexpr uint32_t kIdesc = umma_idesc_f16(2 * BM, BN);
constexpr int kMaxKb = 8;                     // operand K <= 512 (m <= 509 with the 3 norm columns)

struct Params {
  const float* a_norms;
  const uint32_t* endmask;
  const int64_t* seg_offsets;
  const int32_t* range_seg;
  const float* scale;
  float* Z;
  int64_t z_panel;
  int64_t seg_base;  // column c = seg_offsets[s] - seg_base
  int64_t b_rows;
  int z_shift;       // Z panel width = 1 << z_shift segments
  int a_rows;
  int n_mpairs;      // 256-row A tiles
  int n_ranges;
  int n_kb;
  int n_kmma;
  int stages;
};

// shared-memory carve-up; identical offsets in both CTAs of a pair
struct Smem {
  uint32_t A, B;       // shared-window addresses (1024-aligned)
  uint64_t* bars;      // a_full, a_empty, b_full[S], b_empty[S], t_full[2], t_empty[2]
  uint64_t* hand;      // [2 dirs][4 quarters][2 parities] carry hand-off barriers
  float* carry;        // [2 dirs][4 quarters][2 parities][32] running minima
  uint32_t* tmem_slot;
};

constexpr int kHandBars = 2 * 4 * 2;

size_t smem_bytes(int n_kb, int stages) {
  return 1024 + (size_t)n_kb * A_KB_BYTES + (size_t)stages * B_STAGE_BYTES + (2 + 2 * stages + 4) * 8 +
         kHandBars * 8 + kHandBars * 32 * 4 + 16;
}

// ---------------------------------------------------------------------------
// epilogue helpers: branch-free minima over register ranges (static indices)
// ---------------------------------------------------------------------------
constexpr float kInf = __builtin_huge_valf();

__device__ __forceinline__ float fmin3(float a, float b, float c) {
  float r;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));  // FMNMX3 on sm_100a
  return r;
}

template <int A, int B>
struct RangeMin {  // min(v[A..B]) as a balanced ternary tree of 3-input mins (B >= A)
  __device__ __forceinline__ static float run(const float (&v)[32]) {
    constexpr int n = B - A + 1;
    if constexpr (n == 1) {
      return v[A];
    } else if constexpr (n == 2) {
      return fminf(v[A], v[B]);
    } else {
      constexpr int m1 = A + n / 3 - 1 + (n % 3 > 0 ? 1 : 0);
      constexpr int m2 = m1 + n / 3 + (n % 3 > 1 ? 1 : 0);
      return fmin3(RangeMin<A, m1>::run(v), RangeMin<m1 + 1, m2>::run(v), RangeMin<m2 + 1, B>::run(v));
    }
  }
};

// exactly one segment end at column P of the chunk: pre = min(v[0..P]), suf = min(v[P+1..31])
template <int P>
__device__ __forceinline__ void split_at(const float (&v)[32], float& pre, float& suf) {
  pre = RangeMin<0, P>::run(v);
  if constexpr (P < 31) {
    suf = RangeMin<P + 1, 31>::run(v);
  } else {
    suf = kInf;
  }
}

template <int P = 0>
__device__ __forceinline__ void split_switch(int p, const float (&v)[32], float& pre, float& suf) {
  if constexpr (P < 32) {
    if (p == P) {
      split_at<P>(v, pre, suf);
      return;
    }
    split_switch<P + 1>(p, v, pre, suf);
  }
}

__device__ __forceinline__ float masked_min(const float (&v)[32], uint32_t sel) {
  float t[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) t[j] = ((sel >> j) & 1u) ? v[j] : kInf;
  return RangeMin<0, 31>::run(t);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    phase1_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                  const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // keep every pointer derived from smem_raw so the compiler emits shared-space accesses
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  Smem sm;
  sm.A = smem_u32(base);
  sm.B = sm.A + p.n_kb * A_KB_BYTES;
  uint8_t* tail = base + p.n_kb * A_KB_BYTES + p.stages * B_STAGE_BYTES;
  sm.bars = reinterpret_cast<uint64_t*>(tail);
  sm.hand = sm.bars + 2 + 2 * p.stages + 4;
  sm.carry = reinterpret_cast<float*>(sm.hand + kHandBars);
  sm.tmem_slot = reinterpret_cast<uint32_t*>(sm.carry + kHandBars * 32);

  uint64_t* a_full = sm.bars + 0;   // leader: A tiles of both CTAs landed
  uint64_t* a_empty = sm.bars + 1;  // both: the unit's MMAs retired (commit multicast)
  uint64_t* b_full = sm.bars + 2;   // leader: B halves of both CTAs landed
  uint64_t* b_empty = sm.bars + 2 + p.stages;  // both: stage consumed (commit multicast)
  uint64_t* t_full = sm.bars + 2 + 2 * p.stages;  // both: accumulator ready (commit multicast)
  uint64_t* t_empty = sm.bars + 4 + 2 * p.stages;  // leader: 8 epilogue warps drained it

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int64_t pair = blockIdx.x >> 1;
  const int64_t n_pairs = gridDim.x >> 1;

  if (warp == kProducerWarp && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    mbar_init(a_full, 1);
    mbar_init(a_empty, 1);
    for (int i = 0; i < p.stages; ++i) {
      mbar_init(b_full + i, 1);
      mbar_init(b_empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(t_full + i, 1);
      mbar_init(t_empty + i, 2 * kEpiWarps);
    }
    for (int i = 0; i < kHandBars; ++i) mbar_init(sm.hand + i, 1);
    fence_mbar_init();
  }
  if (warp == kAllocWarp) {
    tmem_alloc_2sm(sm.tmem_slot, 512);
    tmem_relinquish_2sm();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *sm.tmem_slot;

  const int64_t n_units = (int64_t)p.n_ranges * p.n_mpairs;

  if (warp == kProducerWarp) {
    // ============================ TMA producer (both CTAs) ============================
    if (lane == 0) {
      const uint64_t pol_a = l2_policy_evict_last();    // A tiles are re-read by every range
      const uint64_t pol_b = l2_policy_evict_normal();  // B ranges are shared by concurrent pairs
      const uint32_t a_full_l = mapa_shared(smem_u32(a_full), 0);
      const uint32_t b_full_l = mapa_shared(smem_u32(b_full), 0);
      uint32_t stage = 0, phase = 0, a_phase = 0;
      int64_t b_loads = 0;
      for (int64_t u = pair; u < n_units; u += n_pairs) {
        const int range = (int)(u / p.n_mpairs);
        const int mp = (int)(u % p.n_mpairs);
        const int s0 = p.range_seg[range], s1 = p.range_seg[range + 1];
        if (s0 == s1) continue;
        const int64_t c_begin = p.seg_offsets[s0] - p.seg_base, c_end = p.seg_offsets[s1] - p.seg_base;
        mbar_wait(a_empty, a_phase ^ 1);
        a_phase ^= 1;
        if (leader) mbar_expect_tx(a_full, 2 * p.n_kb * A_KB_BYTES);
        for (int kb = 0; kb < p.n_kb; ++kb)
          tma_load_2d_2sm(&tmA, a_full_l, smem_raw + (sm.A - smem_u32(smem_raw)) + kb * A_KB_BYTES, kb * BK,
                          mp * 2 * BM + (int)rank * BM, pol_a);
        for (int64_t c0 = c_begin; c0 < c_end; c0 += BN) {
          for (int kb = 0; kb < p.n_kb; ++kb) {
            mbar_wait(b_empty + stage, phase ^ 1);
#if LCRW_EPI_MODE >= 3
            if (b_loads >= p.stages) {  // experiment: ring filled once, then no more B traffic
              if (leader) mbar_arrive(b_full + stage);
            } else
#endif
            {
              if (leader) mbar_expect_tx(b_full + stage, 2 * B_STAGE_BYTES);
              tma_load_2d_2sm(&tmB, b_full_l + stage * 8,
                              smem_raw + (sm.B - smem_u32(smem_raw)) + stage * B_STAGE_BYTES, kb * BK,
                              (int32_t)(c0 + rank * BN_HALF), pol_b);
            }
            ++b_loads;
            if (++stage == (uint32_t)p.stages) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ============================ MMA issuer (leader CTA) =============================
    // The whole warp walks the loop (warp-uniform state); one elected lane issues.
    if (leader) {
      uint32_t stage = 0, phase = 0, a_phase = 0, acc = 0, acc_phase = 0;
      const uint64_t a_desc0 = umma_desc_sw128(sm.A);
      const uint64_t b_desc0 = umma_desc_sw128(sm.B);
      const int last_nk = p.n_kmma - 4 * (p.n_kb - 1);  // MMAs in the last K block (1..4)
      for (int64_t u = pair; u < n_units; u += n_pairs) {
        const int range = (int)(u / p.n_mpairs);
        const int s0 = p.range_seg[range], s1 = p.range_seg[range + 1];
        if (s0 == s1) continue;
        const int64_t c_begin = p.seg_offsets[s0] - p.seg_base, c_end = p.seg_offsets[s1] - p.seg_base;
        mbar_wait(a_full, a_phase);
        a_phase ^= 1;
        tc_fence_after();
        for (int64_t c0 = c_begin; c0 < c_end; c0 += BN) {
#if LCRW_EPI_MODE < 4
          mbar_wait(t_empty + acc, acc_phase ^ 1);
#endif
          tc_fence_after();
          const uint32_t d_tmem = tmem + acc * BN;
          for (int kb = 0; kb < p.n_kb; ++kb) {
            mbar_wait(b_full + stage, phase);
            tc_fence_after();
            // descriptor start-address field counts 16-byte units: +2 per 32-byte K step
            const uint64_t ad = a_desc0 + (uint64_t)(kb * (A_KB_BYTES >> 4));
            const uint64_t bd = b_desc0 + (uint64_t)(stage * (B_STAGE_BYTES >> 4));
            const int nk = kb == p.n_kb - 1 ? last_nk : 4;
            umma_f16_2sm_elect(d_tmem, ad, bd, kIdesc, kb != 0);
            if (nk > 1) umma_f16_2sm_elect(d_tmem, ad + 2, bd + 2, kIdesc, 1);
            if (nk > 2) umma_f16_2sm_elect(d_tmem, ad + 4, bd + 4, kIdesc, 1);
            if (nk > 3) umma_f16_2sm_elect(d_tmem, ad + 6, bd + 6, kIdesc, 1);
            umma_commit_2sm_mc_elect(b_empty + stage, 0x3);  // frees the stage in both CTAs
            if (++stage == (uint32_t)p.stages) {
              stage = 0;
              phase ^= 1;
            }
          }
          umma_commit_2sm_mc_elect(t_full + acc, 0x3);  // accumulator ready in both CTAs' TMEM
          acc ^= 1;
          if (acc == 0) acc_phase ^= 1;
        }
        umma_commit_2sm_mc_elect(a_empty, 0x3);  // A tiles reusable once the unit's MMAs retire
      }
    }
  } else if (warp < kEpiWarps) {
    // ============================ epilogue (both CTAs) ================================
    // Warp (quarter q, half h) owns TMEM lanes [32q, 32q+32) and columns [128h, 128h+128)
    // of every tile.  Segment minima that straddle halves are stitched with a carry
    // hand-off: half 0 of tile t -> half 1 of tile t (dir 0), half 1 of tile t -> half 0
    // of tile t+1 (dir 1).  A half that contains a segment end publishes its tail
    // minimum immediately and only waits for its predecessor to emit its head segment.
    const int quarter = warp & 3;  // TMEM lane quarter accessible to this warp
    const int half = warp >> 2;
    const float inv_scale = p.scale[1];
    const uint32_t t_empty_l = mapa_shared(smem_u32(t_empty), 0);
    const int zs = p.z_shift;
    const int64_t zmask = (1ll << zs) - 1;
    auto hbar = [&](int dir, int par) { return sm.hand + (dir * 4 + quarter) * 2 + par; };
    auto hslot = [&](int dir, int par) { return sm.carry + ((dir * 4 + quarter) * 2 + par) * 32; };

    // tile iterator over this pair's units (skips empty ranges)
    int64_t u = pair - n_pairs, c_begin = 0, c_end = 0, c0 = 0;
    auto next_tile = [&](int64_t& uu, int64_t& cb, int64_t& ce, int64_t& cc) -> int {
      // returns 0 = done, 1 = same unit, 2 = new unit
      if (uu >= 0 && cc + BN < ce) {
        cc += BN;
        return 1;
      }
      for (uu += n_pairs; uu < n_units; uu += n_pairs) {
        const int range = (int)(uu / p.n_mpairs);
        const int s0 = p.range_seg[range], s1 = p.range_seg[range + 1];
        if (s0 == s1) continue;
        cb = p.seg_offsets[s0] - p.seg_base;
        ce = p.seg_offsets[s1] - p.seg_base;
        cc = cb;
        return 2;
      }
      return 0;
    };
    // a tile's segment-end bits: lane i < 8 holds the word of columns [32 i, 32 i + 32)
    auto fetch_mask = [&](int64_t cc) -> uint32_t {
      uint32_t w = 0;
      if (lane < BN / 32) {
        const int64_t bit = cc + lane * 32;
        const uint32_t lo = __ldg(p.endmask + (bit >> 5));
        const uint32_t hi = __ldg(p.endmask + (bit >> 5) + 1);
        w = __funnelshift_r(lo, hi, (uint32_t)(bit & 31));
      }
      return w;
    };

    int kind = next_tile(u, c_begin, c_end, c0);
    uint32_t pm = kind ? fetch_mask(c0) : 0u;
    uint32_t acc = 0, acc_phase = 0, tcount = 0;
    bool valid = false;
    float nE = 0.f;
    float* zrow = p.Z;
    int64_t s_tile = 0;
    while (kind) {
      if (kind == 2) {  // first tile of a unit
        const int mp = (int)(u % p.n_mpairs);
        const int range = (int)(u / p.n_mpairs);
        const int row = mp * 2 * BM + (int)rank * BM + quarter * 32 + lane;
        valid = row < p.a_rows;
        nE = valid ? __ldg(p.a_norms + row) : 0.f;
        zrow = p.Z + ((int64_t)row << zs);
        s_tile = p.range_seg[range];
      }
      const bool unit_start = kind == 2;
      const int ncols = (int)min((int64_t)BN, c_end - c0);
      // segment-end bits of this tile, restricted to its columns
      uint32_t wmask = __shfl_sync(0xffffffffu, pm, lane & 7);
      {
        const int lim = ncols - (lane & 7) * 32;
        wmask = lim >= 32 ? wmask : (lim <= 0 ? 0u : (wmask & ((1u << lim) - 1u)));
      }
      const int ends0 = __popc(__shfl_sync(0xffffffffu, wmask, 0)) + __popc(__shfl_sync(0xffffffffu, wmask, 1)) +
                        __popc(__shfl_sync(0xffffffffu, wmask, 2)) + __popc(__shfl_sync(0xffffffffu, wmask, 3));
      const int ends1 = __popc(__shfl_sync(0xffffffffu, wmask, 4)) + __popc(__shfl_sync(0xffffffffu, wmask, 5)) +
                        __popc(__shfl_sync(0xffffffffu, wmask, 6)) + __popc(__shfl_sync(0xffffffffu, wmask, 7));
      // prefetch the next tile's segment bits while this tile is processed
      int64_t nu = u, ncb = c_begin, nce = c_end, nc0 = c0;
      const int nkind = next_tile(nu, ncb, nce, nc0);
      if (nkind) pm = fetch_mask(nc0);

      int64_t s = s_tile + (half ? ends0 : 0);  // first segment ending in (or after) my half
      const int64_t s_head = s;
      float head = kInf, run = kInf;
      bool have_end = false;
      auto emit = [&](int64_t seg, float segmin) {
        if (valid) {
          float d;
          asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(d) : "f"(fmaxf(segmin + nE, 0.f)));
          zrow[(seg >> zs) * p.z_panel + (seg & zmask)] = d * inv_scale;
        }
      };
      // segment end inside my half: the first one closes the head (emitted after the hand-off)
      auto close = [&](float segmin) {
        if (!have_end) {
          head = segmin;
          have_end = true;
        } else {
          emit(s, segmin);
        }
        ++s;
      };

      const int my_cols = min(BN_HALF, ncols - half * BN_HALF);
      mbar_wait(t_full + acc, acc_phase);
      tc_fence_after();
      const uint32_t t_base = tmem + ((uint32_t)(quarter * 32) << 16) + acc * BN + half * BN_HALF;
#pragma unroll 1
      for (int ch = 0; ch < BN_HALF / 32; ++ch) {
        if (ch * 32 >= my_cols) break;
        uint32_t raw[32];
#if LCRW_EPI_MODE >= 2
        if (ch >= 0) { run = fminf(run, (float)ch); continue; }
#endif
#if LCRW_EPI_MODE == 1
        tmem_ld_32x32b_x32(t_base + ch * 32, raw);
        tmem_wait_ld();
        run = fminf(run, fminf(__uint_as_float(raw[0]), __uint_as_float(raw[31])));
        continue;
#endif
        tmem_ld_32x32b_x32(t_base + ch * 32, raw);
        tmem_wait_ld();

        // the accumulator already holds v_j = |B_j|^2 - 2 A.B_j (norm columns folded into K)
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(raw[j]);
        const int lim = my_cols - ch * 32;
        uint32_t mask = __shfl_sync(0xffffffffu, wmask, half * 4 + ch);
        if (lim < 32) {  // columns >= lim belong to the next range
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j >= lim) v[j] = kInf;
        }
        const int nb_ends = __popc(mask);
        if (nb_ends == 0) {
          run = fminf(run, RangeMin<0, 31>::run(v));
        } else if (nb_ends == 1) {
          float pre, suf;
          split_switch(__ffs(mask) - 1, v, pre, suf);
          close(fminf(run, pre));
          run = suf;
        } else {
          int start = 0;
          while (mask) {
            const int e = __ffs(mask) - 1;
            mask &= mask - 1u;
            const uint32_t upto = e == 31 ? 0xFFFFFFFFu : ((2u << e) - 1u);
            close(fminf(run, masked_min(v, upto & (0xFFFFFFFFu << start))));
            run = kInf;
            start = e + 1;
          }
          if (start < 32) run = masked_min(v, 0xFFFFFFFFu << start);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster_relaxed(t_empty_l + acc * 8);  // leader's t_empty[acc]

      // ---- carry hand-off: pred -> me (dir = 1 - half), me -> succ (dir = half) ----
      const int par = tcount & 1;
      const int in_dir = half ? 0 : 1;
      const int in_par = half ? par : (par ^ 1);          // half 0 reads tile t-1's half 1
      const uint32_t in_phase = half ? (tcount >> 1) & 1 : ((tcount - 1) >> 1) & 1;
      const bool has_pred = half ? true : (tcount > 0);
      auto publish = [&](float carry_out) {
        float* slot = hslot(half, par);
        slot[lane] = carry_out;
        __syncwarp();
        if (lane == 0) mbar_arrive(hbar(half, par));
      };
      auto receive = [&]() -> float {
        if (!has_pred) return kInf;
        mbar_wait(hbar(in_dir, in_par), in_phase);
        const float c = hslot(in_dir, in_par)[lane];
        return (half == 0 && unit_start) ? kInf : c;  // a unit starts with no open segment
      };
      // Half 0 publishes before receiving (its tail does not depend on the carry);
      // half 1 always receives first, which keeps every hand-off barrier at most one
      // phase ahead of its consumer (an mbarrier parity wait cannot skip a phase).
      if (half == 0 && have_end) {
        publish(run);
        emit(s_head, fminf(receive(), head));
      } else {
        const float cin = receive();
        if (have_end) {
          emit(s_head, fminf(cin, head));
          publish(run);
        } else {
          publish(fminf(cin, run));
        }
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
      ++tcount;
      s_tile += ends0 + ends1;
      u = nu;
      c_begin = ncb;
      c_end = nce;
      c0 = nc0;
      kind = nkind;
    }
    // drain: half 0 consumes the last hand-off of half 1 so no arrival is left pending
    if (half == 0 && tcount > 0) {
      const int lp = (tcount - 1) & 1;
      mbar_wait(hbar(1, lp), ((tcount - 1) >> 1) & 1);
    }
  }

  __syncwarp();  // reconverge single-lane roles before the aligned cluster barrier
  tc_fence_before();
  cluster_sync();
  if (warp == kAllocWarp) {
    tc_fence_after();
    tmem_dealloc_2sm(tmem, 512);
  }
}

// ---------------------------------------------------------------------------
// host side: tensor maps via the driver entry point (no -lcuda link needed)
// ---------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

int make_map(CUtensorMap* map, const void* base, int64_t rows, int kp, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable (driver too old?)");
    return LCRW_ERR_CUDA;
  }
  cuuint64_t dims[2] = {(cuuint64_t)kp, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)kp * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d) rows=%lld kp=%d", (int)r, (long long)rows, kp);
    return LCRW_ERR_CUDA;
  }
  return LCRW_OK;
}

}  // namespace p1
}  // namespace lcrw

namespace lcrw {
namespace p1 {

int launch(const uint16_t* A, const float* a_norms, int64_t a_rows, const uint16_t* B, int64_t b_rows, int m, int kp, const int64_t* seg_offsets, int64_t seg_base, int64_t n_seg,
           const uint32_t* endmask, const int32_t* range_seg, int64_t n_ranges, const float* scale, float* Z,
           int64_t z_panel, int z_shift, cudaStream_t stream, const char* tag) {
  LCRW_REQUIRE(m > 0 && kp == lcrw_padded_dim(m), "lcrw_phase1: kp must be lcrw_padded_dim(K)");
  LCRW_REQUIRE(a_rows >= 0 && a_rows < (1ll << 31) && b_rows >= 0 && b_rows < (1ll << 31),
               "lcrw_phase1: row counts must fit in int32");
  LCRW_REQUIRE(n_seg >= 0 && n_ranges >= 1, "lcrw_phase1: bad segment plan");
  LCRW_REQUIRE(z_shift >= 0 && z_shift <= 10, "lcrw_phase1: z_shift out of range");
  LCRW_REQUIRE(z_panel >= (a_rows << z_shift), "lcrw_phase1: z_panel must be >= a_rows << z_shift");
  if (a_rows == 0 || n_seg == 0) return LCRW_OK;
  LCRW_REQUIRE(A && a_norms && B && seg_offsets && endmask && range_seg && scale && Z,
               "lcrw_phase1: null pointer");
  LCRW_REQUIRE((reinterpret_cast<uintptr_t>(A) & 15) == 0 && (reinterpret_cast<uintptr_t>(B) & 15) == 0,
               "lcrw_phase1: operands must be 16-byte aligned");
  const int n_kb = kp / BK;
  if (n_kb > kMaxKb) {
    set_error("lcrw_phase1: operand K = %d (embedding dimension + 3 norm columns) > %d unsupported", m,
              kMaxKb * BK);
    return LCRW_ERR_UNSUPPORTED;
  }
  // A K-blocks + B stages within ~208 KB of shared memory
  const int stages = n_kb <= 5 ? 8 : 13 - n_kb;
  Params p;
  p.a_norms = a_norms;
  p.endmask = endmask;
  p.seg_offsets = seg_offsets;
  p.range_seg = range_seg;
  p.scale = scale;
  p.Z = Z;
  p.z_panel = z_panel;
  p.seg_base = seg_base;
  p.b_rows = b_rows;
  p.z_shift = z_shift;
  p.a_rows = (int)a_rows;
  p.n_mpairs = (int)ceil_div(a_rows, 2 * BM);
  p.n_ranges = (int)n_ranges;
  p.n_kb = n_kb;
  p.n_kmma = (m + 15) / 16;
  p.stages = stages;

  CUtensorMap tmA, tmB;
  int st = make_map(&tmA, A, a_rows, kp, BM);
  if (st) return st;
  st = make_map(&tmB, B, b_rows, kp, BN_HALF);
  if (st) return st;

  const size_t smem = smem_bytes(n_kb, stages);
  static bool attr_set = false;
  if (!attr_set) {
    size_t mx = smem_bytes(5, 8);
    for (int kb = 6; kb <= kMaxKb; ++kb)
      if (smem_bytes(kb, 13 - kb) > mx) mx = smem_bytes(kb, 13 - kb);
    cudaError_t e = cudaFuncSetAttribute(phase1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(phase1_kernel)");
    attr_set = true;
  }
  const int64_t n_units = (int64_t)n_ranges * p.n_mpairs;
  const int64_t pairs = sm_count() / 2;
  const int grid = 2 * (int)(n_units < pairs ? n_units : pairs);
  ProfScope prof(stream, tag);
  phase1_kernel<<<grid, kThreads, smem, stream>>>(tmA, tmB, p);
  LCRW_CHECK_LAUNCH("phase1_kernel");
  return LCRW_OK;
}

}  // namespace p1
}  // namespace lcrw

extern "C" int lcrw_phase1(const uint16_t* A, const float* a_norms, int64_t a_rows, const uint16_t* B,
                           int64_t b_rows, int m, int kp, const int64_t* seg_offsets,
                           int64_t seg_base, int64_t n_seg, const uint32_t* endmask, const int32_t* range_seg,
                           int64_t n_ranges, const float* scale, float* Z, int64_t z_panel, int z_shift,
                           void* stream) {
  return lcrw::p1::launch(A, a_norms, a_rows, B, b_rows, m, kp, seg_offsets, seg_base, n_seg, endmask,
                          range_seg, n_ranges, scale, Z, z_panel, z_shift, lcrw::as_stream(stream), "phase1");
}
