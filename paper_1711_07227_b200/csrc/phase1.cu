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
// Work unit = (pair of 128-row m-tiles, two consecutive column ranges of
// ~range_cols B rows each, bounded by segment boundaries).  The two ranges of a
// unit ("halves") are interleaved tile by tile and each owns one of the two TMEM
// accumulator buffers: half h's tiles always land in buffer h and are reduced by
// epilogue warp group h, so a segment's running minimum never leaves the
// registers of the warp that reduces it (ranges never cut a segment), every Z
// entry is written exactly once, and there is no atomic, initialisation pass
// or cross-warp hand-off.
//
// Warp roles (352 threads per CTA): w0..w7 epilogue (TMEM lane quarter = warp % 4,
// accumulator buffer / unit half = warp / 4, one A row per thread), w8 TMA
// producer, w9 MMA issuer (leader CTA only), w10 TMEM allocator.
#include <cstdio>

#include "common.cuh"

namespace lcrw {
namespace p1 {

#ifdef LCRW_P1_STATS
// experiment instrumentation (variants/build_stats.sh; not in the shipped build): cycle
// counters [0] epilogue wait t_full, [1] epilogue tile work, [3] epilogue tiles,
// [4] MMA wait t_empty, [5] MMA wait b_full, [6] MMA tiles
__device__ unsigned long long g_p1_stats[8];
#endif

constexpr int BM = 128;                       // A rows per CTA (TMEM lanes); the pair covers 256
constexpr int BN = 256;                       // B rows per pair tile (MMA N); 128 staged per CTA
constexpr int BN_HALF = BN / 2;
constexpr int BK = 64;                        // f16 elements per K block (128 B rows)
constexpr int A_KB_BYTES = BM * BK * 2;       // 16 KB
constexpr int B_STAGE_BYTES = BN_HALF * BK * 2;  // 16 KB per CTA
constexpr int kEpiWarps = 8;                  // two groups (accumulator buffers) x four TMEM lane quarters
// Warp roles.  The schedulers favour higher warp ids, so the single-lane TMA and
// MMA issuers sit above the epilogue warps and are never starved by them.
constexpr int kProducerWarp = kEpiWarps;      // 8
constexpr int kMmaWarp = kEpiWarps + 1;       // 9
constexpr int kAllocWarp = kEpiWarps + 2;     // 10
constexpr int kThreads = 32 * (kEpiWarps + 3);
constexpr uint32_t kIdesc = umma_idesc_f16(2 * BM, BN);
constexpr int kMaxKb = 8;                     // resident A: operand K <= 512 (m <= 509 with the 3 norm columns)
constexpr int kMaxKbStream = 64;              // streamed A (K > 512): operand K <= 4096
constexpr int kStreamStages = 6;              // streamed A: ring stages of (A + B) K blocks, 32 KB each

// output forms of the epilogue
enum ZMode : int {
  kZPanels = 0,     // f32 Z[(s >> zs) * z_panel + (row << zs) + (s & (zw-1))] (segment panels)
  kZPanelsKey = 1,  // the same, values rounded through the 21-bit key (reverse direction, GEMM form)
  kZTable = 2,      // packed 21-bit distance table (kTableChunk-word chunks, kTableRowBytes per
                    // segment = vocabulary word; z_panel = bytes per chunk; common.cuh)
};

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
  const int32_t* b_ids;  // gather mode: B row c is operand row b_ids[c] (TMA gather4); NULL = rows in order
  int32_t b_oob;         // gather mode: a row index past the operand table (zero-filled padding rows)
  int z_shift;       // Z panel width = 1 << z_shift segments
  int z_mode;        // ZMode: Z layout / value form of the output
  int a_rows;
  int n_mpairs;      // 256-row A tiles
  int n_ranges;      // column ranges; a work unit takes two consecutive ones
  int n_kb;
  int n_kmma;
  int stages;
  int a_stream;      // 1: A K blocks streamed through the ring with B's (operand K > 512)
};

// shared-memory carve-up; identical offsets in both CTAs of a pair
struct Smem {
  uint32_t A, B;       // shared-window addresses (1024-aligned)
  uint64_t* bars;      // a_full, a_empty, b_full[S], b_empty[S], t_full[2], t_empty[2]
  uint32_t* tmem_slot;
};

size_t smem_bytes(int n_kb, int stages, bool a_stream = false) {
  if (a_stream)  // no resident A; each stage holds an A K block followed by a B K block
    return 1024 + (size_t)stages * (A_KB_BYTES + B_STAGE_BYTES) + (2 + 2 * stages + 4) * 8 + 16;
  return 1024 + (size_t)n_kb * A_KB_BYTES + (size_t)stages * B_STAGE_BYTES + (2 + 2 * stages + 4) * 8 + 16;
}

// a work unit's two halves: half h = columns [c[h], c[h+1]), first segment s[h] (scalars, no
// dynamically indexed arrays, so the struct stays in registers)
struct Unit {
  int64_t c0, c1, c2;
  int s0, s1;
  int n0, n1;  // BN-column tiles per half
  __device__ __forceinline__ int64_t cb(int h) const { return h ? c1 : c0; }
  __device__ __forceinline__ int64_t ce(int h) const { return h ? c2 : c1; }
  __device__ __forceinline__ int sb(int h) const { return h ? s1 : s0; }
};

__device__ __forceinline__ bool unit_plan(const Params& p, int64_t u, Unit& U) {
  const int rp = (int)(u / p.n_mpairs);
  const int r0 = 2 * rp, r1 = min(2 * rp + 1, p.n_ranges), r2 = min(2 * rp + 2, p.n_ranges);
  const int s0 = p.range_seg[r0], s1 = p.range_seg[r1], s2 = p.range_seg[r2];
  if (s0 == s2) return false;
  U.c0 = p.seg_offsets[s0] - p.seg_base;
  U.c1 = p.seg_offsets[s1] - p.seg_base;
  U.c2 = p.seg_offsets[s2] - p.seg_base;
  U.s0 = s0;
  U.s1 = s1;
  U.n0 = (int)((U.c1 - U.c0 + BN - 1) / BN);
  U.n1 = (int)((U.c2 - U.c1 + BN - 1) / BN);
  return true;
}

// interleaved tile order of a unit: i -> (half, tile index within the half)
__device__ __forceinline__ void unit_tile(const Unit& U, int i, int& h, int& k) {
  const int both = 2 * min(U.n0, U.n1);
  if (i < both) {
    h = i & 1;
    k = i >> 1;
  } else {
    h = U.n0 > U.n1 ? 0 : 1;
    k = (both >> 1) + (i - both);
  }
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

// min(run, v[0..31]) in 17 min instructions (16 three-input): 33 -> 11 -> 4 -> 2 -> 1
__device__ __forceinline__ float chunk_min(float run, const float (&v)[32]) {
  const float a0 = fmin3(run, v[0], v[1]), a1 = fmin3(v[2], v[3], v[4]), a2 = fmin3(v[5], v[6], v[7]);
  const float a3 = fmin3(v[8], v[9], v[10]), a4 = fmin3(v[11], v[12], v[13]), a5 = fmin3(v[14], v[15], v[16]);
  const float a6 = fmin3(v[17], v[18], v[19]), a7 = fmin3(v[20], v[21], v[22]), a8 = fmin3(v[23], v[24], v[25]);
  const float a9 = fmin3(v[26], v[27], v[28]), a10 = fmin3(v[29], v[30], v[31]);
  const float b0 = fmin3(a0, a1, a2), b1 = fmin3(a3, a4, a5), b2 = fmin3(a6, a7, a8), b3 = fminf(a9, a10);
  return fminf(fmin3(b0, b1, b2), b3);
}

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

#include "split_ptx.inc"

// exactly one segment end at the warp-uniform column p: one indirect branch through a
// 32-entry PTX jump table (gen_split.py), each target a pair of 3-input-min trees
__device__ __forceinline__ void split_switch(int p, const float (&v)[32], float& pre, float& suf) {
  asm(LCRW_SPLIT_PTX
      : "=f"(pre), "=f"(suf)
      : "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]),
        "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]),
        "f"(v[17]), "f"(v[18]), "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]),
        "f"(v[25]), "f"(v[26]), "f"(v[27]), "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31]), "r"(p));
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
  // resident A: [A K blocks][B stages]; streamed A: [stage: A K block, B K block] x stages
  const int a_res_kb = p.a_stream ? 0 : p.n_kb;
  const uint32_t stage_bytes = p.a_stream ? A_KB_BYTES + B_STAGE_BYTES : B_STAGE_BYTES;
  const uint32_t b_in_stage = p.a_stream ? A_KB_BYTES : 0;
  sm.A = smem_u32(base);
  sm.B = sm.A + a_res_kb * A_KB_BYTES;
  uint8_t* tail = base + a_res_kb * A_KB_BYTES + p.stages * stage_bytes;
  sm.bars = reinterpret_cast<uint64_t*>(tail);
  sm.tmem_slot = reinterpret_cast<uint32_t*>(sm.bars + 2 + 2 * p.stages + 4);

  uint64_t* a_full = sm.bars + 0;   // leader: A tiles of both CTAs landed
  uint64_t* a_empty = sm.bars + 1;  // both: the unit's MMAs retired (commit multicast)
  uint64_t* b_full = sm.bars + 2;   // leader: B halves of both CTAs landed
  uint64_t* b_empty = sm.bars + 2 + p.stages;  // both: stage consumed (commit multicast)
  uint64_t* t_full = sm.bars + 2 + 2 * p.stages;  // both: accumulator ready (commit multicast)
  uint64_t* t_empty = sm.bars + 4 + 2 * p.stages;  // leader: the buffer's 4 epilogue warps (x2 CTAs) drained it

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
      mbar_init(t_empty + i, kEpiWarps);  // 4 warps per buffer in each of the 2 CTAs
    }
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

  const int64_t n_units = (int64_t)((p.n_ranges + 1) / 2) * p.n_mpairs;

  if (warp == kProducerWarp) {
    // ============================ TMA producer (both CTAs) ============================
    // The whole warp walks the loop; lane 0 issues tile loads, every lane issues its
    // 4-row TMA gathers in gather mode.
    {
      const uint64_t pol_a = l2_policy_evict_last();    // A tiles are re-read by every range
      const uint64_t pol_b = l2_policy_evict_normal();  // B ranges are shared by concurrent pairs
      const uint32_t a_full_l = mapa_shared(smem_u32(a_full), 0);
      const uint32_t b_full_l = mapa_shared(smem_u32(b_full), 0);
      uint32_t stage = 0, phase = 0, a_phase = 0;
      const uint32_t tx_bytes = 2 * B_STAGE_BYTES + (p.a_stream ? 2 * A_KB_BYTES : 0);  // both CTAs' halves
      for (int64_t u = pair; u < n_units; u += n_pairs) {
        Unit U;
        if (!unit_plan(p, u, U)) continue;
        const int mp = (int)(u % p.n_mpairs);
        const int a_row = mp * 2 * BM + (int)rank * BM;
        if (!p.a_stream) mbar_wait(a_empty, a_phase ^ 1);
        a_phase ^= 1;
        if (lane == 0 && !p.a_stream) {
          if (leader) mbar_expect_tx(a_full, 2 * p.n_kb * A_KB_BYTES);
          for (int kb = 0; kb < p.n_kb; ++kb)
            tma_load_2d_2sm(&tmA, a_full_l, smem_raw + (sm.A - smem_u32(smem_raw)) + kb * A_KB_BYTES, kb * BK,
                            mp * 2 * BM + (int)rank * BM, pol_a);
        }
        const int n_tiles = U.n0 + U.n1;
        for (int i = 0; i < n_tiles; ++i) {
          int h, k;
          unit_tile(U, i, h, k);
          const int64_t c0 = U.cb(h) + (int64_t)k * BN;
          // gather mode: lane l owns B rows 4l .. 4l+3 of this CTA's half tile
          int32_t g0 = 0, g1 = 0, g2 = 0, g3 = 0;
          if (p.b_ids) {
            const int64_t cb = c0 + rank * BN_HALF + 4 * lane;
            auto id_at = [&](int64_t c) -> int32_t { return c < p.b_rows ? __ldg(p.b_ids + c) : p.b_oob; };
            g0 = id_at(cb);
            g1 = id_at(cb + 1);
            g2 = id_at(cb + 2);
            g3 = id_at(cb + 3);
          }
          for (int kb = 0; kb < p.n_kb; ++kb) {
            mbar_wait(b_empty + stage, phase ^ 1);
            uint8_t* const st_ptr = smem_raw + (sm.B - smem_u32(smem_raw)) + stage * stage_bytes;
            // streamed A: this K block of the unit's A rows rides with B's on the stage's
            // barrier (one arrive.expect_tx for both: the barrier expects one arrival)
            if (p.a_stream && lane == 0) tma_load_2d_2sm(&tmA, b_full_l + stage * 8, st_ptr, kb * BK, a_row, pol_a);
            if (p.b_ids) {
              if (leader && lane == 0) mbar_expect_tx(b_full + stage, tx_bytes);
              tma_gather4_2sm(&tmB, b_full_l + stage * 8, st_ptr + b_in_stage + lane * 4 * BK * 2,
                              kb * BK, g0, g1, g2, g3, pol_b);
            } else if (lane == 0) {
              {
                if (leader) mbar_expect_tx(b_full + stage, tx_bytes);
                tma_load_2d_2sm(&tmB, b_full_l + stage * 8, st_ptr + b_in_stage, kb * BK,
                                (int32_t)(c0 + rank * BN_HALF), pol_b);
              }
            }
            __syncwarp();
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
      uint32_t stage = 0, phase = 0, a_phase = 0, e_phase = 0;  // e_phase bit h: t_empty[h] parity
      const uint64_t a_desc0 = umma_desc_sw128(sm.A);
      const uint64_t b_desc0 = umma_desc_sw128(sm.B);
      const int last_nk = p.n_kmma - 4 * (p.n_kb - 1);  // MMAs in the last K block (1..4)
      for (int64_t u = pair; u < n_units; u += n_pairs) {
        Unit U;
        if (!unit_plan(p, u, U)) continue;
        if (!p.a_stream) mbar_wait(a_full, a_phase);
        a_phase ^= 1;
        tc_fence_after();
        const int n_tiles = U.n0 + U.n1;
        for (int i = 0; i < n_tiles; ++i) {
          int h, k;
          unit_tile(U, i, h, k);
#ifdef LCRW_P1_STATS
          const long long _t0 = clock64();
#endif
          mbar_wait(t_empty + h, ((e_phase >> h) & 1) ^ 1);
#ifdef LCRW_P1_STATS
          if (lane == 0) {
            atomicAdd(&g_p1_stats[4], (unsigned long long)(clock64() - _t0));
            atomicAdd(&g_p1_stats[6], 1ull);
          }
#endif
          e_phase ^= 1u << h;
          tc_fence_after();
          const uint32_t d_tmem = tmem + h * BN;
          for (int kb = 0; kb < p.n_kb; ++kb) {
#ifdef LCRW_P1_STATS
            const long long _t1 = clock64();
#endif
            mbar_wait(b_full + stage, phase);
#ifdef LCRW_P1_STATS
            if (lane == 0) atomicAdd(&g_p1_stats[5], (unsigned long long)(clock64() - _t1));
#endif
            tc_fence_after();
            // descriptor start-address field counts 16-byte units: +2 per 32-byte K step
            const uint64_t ad = p.a_stream ? b_desc0 + (uint64_t)(stage * (stage_bytes >> 4))
                                           : a_desc0 + (uint64_t)(kb * (A_KB_BYTES >> 4));
            const uint64_t bd = b_desc0 + (uint64_t)((stage * stage_bytes + b_in_stage) >> 4);
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
          umma_commit_2sm_mc_elect(t_full + h, 0x3);  // accumulator h ready in both CTAs' TMEM
        }
        if (!p.a_stream) umma_commit_2sm_mc_elect(a_empty, 0x3);  // A tiles reusable once the unit's MMAs retire
      }
    }
  } else if (warp < kEpiWarps) {
    // ============================ epilogue (both CTAs) ================================
    // Warp (quarter q, group h) owns TMEM lanes [32q, 32q+32) (= 32 A rows, one per
    // lane) of accumulator buffer h, i.e. of every tile of each unit's half h.  The
    // segment structure is the same for all rows, so every branch below is warp-uniform.
    const int quarter = warp & 3;
    const int grp = warp >> 2;
    const float inv_scale = p.scale[1];
    const uint32_t t_empty_l = mapa_shared(smem_u32(t_empty + grp), 0);
    const int zs = p.z_shift;
    const uint32_t zw = 1u << zs;
    // a tile's segment-end bits: lane i < 8 holds the word of columns [c + 32 i, c + 32 i + 32)
    auto fetch_mask = [&](int64_t c) -> uint32_t {
      uint32_t w = 0;
      if (lane < BN / 32) {
        const int64_t bit = c + lane * 32;
        const uint32_t lo = __ldg(p.endmask + (bit >> 5));
        const uint32_t hi = __ldg(p.endmask + (bit >> 5) + 1);
        w = __funnelshift_r(lo, hi, (uint32_t)(bit & 31));
      }
      return w;
    };
    uint32_t phase = 0;
    for (int64_t u = pair; u < n_units; u += n_pairs) {
      Unit U;
      if (!unit_plan(p, u, U)) continue;
      const int64_t c_lo = U.cb(grp), c_hi = U.ce(grp);
      if (c_lo == c_hi) continue;
      const int mp = (int)(u % p.n_mpairs);
      const int row = mp * 2 * BM + (int)rank * BM + quarter * 32 + lane;
      const bool valid = row < p.a_rows;
      const float nE = valid ? __ldg(p.a_norms + row) : 0.f;
      // output cursor: segment s = U.sb(grp) + emitted so far, at
      //   Z[(s >> zs) * z_panel + (row << zs) + (s & (zw-1))]   (segment panels), or
      //   table bytes: chunk row / 256, row s of 512 bytes, key (row % 256) -- a warp's 32
      //   rows are 64 contiguous bytes of the row
      const int64_t s_first = U.sb(grp);
      float* zq;
      int64_t step, wrap;
      uint32_t s_in = (uint32_t)s_first & (zw - 1);
      uint8_t* zb = nullptr;
      const uint32_t kbase = key16_base(nE);  // the row word's 16-bit key range (reverse direction)
      if (p.z_mode == kZTable) {
        zq = nullptr;
        step = wrap = 0;
        zb = reinterpret_cast<uint8_t*>(p.Z) + ((int64_t)row / kTableChunk) * p.z_panel + s_first * kTableRowBytes +
             (row % kTableChunk) * 2;
      } else {
        zq = p.Z + (s_first >> zs) * p.z_panel + ((int64_t)row << zs) + s_in;
        step = 1;
        wrap = p.z_panel - zw;
      }
      float run = kInf;
      auto emit = [&](float segmin) {
        float d;
        asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(d) : "f"(fmaxf(segmin + nE, 0.f)));
        if (p.z_mode == kZTable) {
          // every lane stores (no branch per emit, so the encodes interleave): rows past a_rows
          // are the last chunk's unused words, inside the table and never read as values
          *reinterpret_cast<uint16_t*>(zb) = (uint16_t)dist_key16(d, kbase);
          zb += kTableRowBytes;
          return;
        }
        if (p.z_mode == kZPanelsKey) d = key16_dist(dist_key16(d, kbase), kbase);
        if (valid) *zq = d * inv_scale;
        zq += step;
        if (++s_in == zw) {
          s_in = 0;
          zq += wrap;
        }
      };
      uint32_t pm = fetch_mask(c_lo);
      for (int64_t c0 = c_lo; c0 < c_hi; c0 += BN) {
        const int ncols = (int)min((int64_t)BN, c_hi - c0);
        uint32_t wmask = pm;
        {
          const int lim = ncols - lane * 32;
          wmask = lim >= 32 ? wmask : (lim <= 0 ? 0u : (wmask & ((1u << lim) - 1u)));
        }
        if (c0 + BN < c_hi) pm = fetch_mask(c0 + BN);  // next tile's bits, latency hidden behind this one
#ifdef LCRW_P1_STATS
        const long long _tw = clock64();
#endif
        mbar_wait(t_full + grp, phase);
#ifdef LCRW_P1_STATS
        const long long _tc = clock64();
        if (lane == 0) {
          atomicAdd(&g_p1_stats[0], (unsigned long long)(_tc - _tw));
          atomicAdd(&g_p1_stats[3], 1ull);
        }
#endif
        tc_fence_after();
        const uint32_t t_base = tmem + ((uint32_t)(quarter * 32) << 16) + grp * BN;
        const int nch = (ncols + 31) >> 5;
#pragma unroll 1
        for (int ch = 0; ch < nch; ++ch) {
          uint32_t raw[32];
          tmem_ld_32x32b_x32(t_base + ch * 32, raw);
          tmem_wait_ld();
          // the accumulator holds v_j = |B_j|^2 - 2 A.B_j (norm columns folded into K)
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(raw[j]);
          uint32_t mask = __shfl_sync(0xffffffffu, wmask, ch);
          if (mask == 0) {
            run = chunk_min(run, v);
          } else if ((mask & (mask - 1u)) == 0) {  // exactly one segment end in the chunk
            float pre, suf;
            split_switch(__ffs(mask) - 1, v, pre, suf);
            emit(fminf(run, pre));
            run = suf;
          } else if (mask == 0xFFFFFFFFu) {  // every column closes a segment (pairwise distances)
            emit(fminf(run, v[0]));
#pragma unroll
            for (int j = 1; j < 32; ++j) emit(v[j]);
            run = kInf;
          } else {
            int start = 0;
            while (mask) {
              const int e = __ffs(mask) - 1;
              mask &= mask - 1u;
              const uint32_t upto = e == 31 ? 0xFFFFFFFFu : ((2u << e) - 1u);
              emit(fminf(run, masked_min(v, upto & (0xFFFFFFFFu << start))));
              run = kInf;
              start = e + 1;
            }
            run = start < 32 ? masked_min(v, 0xFFFFFFFFu << start) : kInf;
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster_relaxed(t_empty_l);  // leader's t_empty[grp]
        phase ^= 1;
#ifdef LCRW_P1_STATS
        if (lane == 0) atomicAdd(&g_p1_stats[1], (unsigned long long)(clock64() - _tc));
#endif
      }
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

int launch(const uint16_t* A, const float* a_norms, int64_t a_rows, const uint16_t* B, int64_t b_rows, int m, int kp,
           const int64_t* seg_offsets, int64_t seg_base, int64_t n_seg, const uint32_t* endmask,
           const int32_t* range_seg, int64_t n_ranges, const float* scale, float* Z, int64_t z_panel, int z_shift,
           cudaStream_t stream, const char* tag, const int32_t* b_ids, int64_t b_table_rows, int z_mode) {
  LCRW_REQUIRE(m > 0 && kp == lcrw_padded_dim(m), "lcrw_phase1: kp must be lcrw_padded_dim(K)");
  LCRW_REQUIRE(a_rows >= 0 && a_rows < (1ll << 31) && b_rows >= 0 && b_rows < (1ll << 31),
               "lcrw_phase1: row counts must fit in int32");
  LCRW_REQUIRE(n_seg >= 0 && n_ranges >= 1, "lcrw_phase1: bad segment plan");
  LCRW_REQUIRE(z_shift >= 0 && z_shift <= 10, "lcrw_phase1: z_shift out of range");
  LCRW_REQUIRE(z_mode == kZTable ? z_panel >= n_seg * kTableRowBytes : z_panel >= (a_rows << z_shift),
               "lcrw_phase1: z_panel must be >= a_rows << z_shift (packed table: n_seg * kTableRowBytes)");
  if (a_rows == 0 || n_seg == 0) return LCRW_OK;
  LCRW_REQUIRE(A && a_norms && B && seg_offsets && endmask && range_seg && scale && Z,
               "lcrw_phase1: null pointer");
  LCRW_REQUIRE((reinterpret_cast<uintptr_t>(A) & 15) == 0 && (reinterpret_cast<uintptr_t>(B) & 15) == 0,
               "lcrw_phase1: operands must be 16-byte aligned");
  const int n_kb = kp / BK;
  if (n_kb > kMaxKbStream) {
    set_error("lcrw_phase1: operand K = %d (embedding dimension + 3 norm columns) > %d unsupported", m,
              kMaxKbStream * BK);
    return LCRW_ERR_UNSUPPORTED;
  }
  // resident A K-blocks + B stages within ~208 KB of shared memory; beyond K = 512 the A
  // K blocks are streamed with B's (each tile re-reads its A rows: more L2->SM bytes,
  // same MMAs)
  const bool a_stream = n_kb > kMaxKb;
  const int stages = a_stream ? kStreamStages : (n_kb <= 5 ? 8 : 13 - n_kb);
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
  p.b_ids = b_ids;
  p.b_oob = (int32_t)b_table_rows;
  p.z_shift = z_shift;
  p.z_mode = z_mode;
  p.a_rows = (int)a_rows;
  p.n_mpairs = (int)ceil_div(a_rows, 2 * BM);
  p.n_ranges = (int)n_ranges;
  p.n_kb = n_kb;
  p.n_kmma = (m + 15) / 16;
  p.stages = stages;
  p.a_stream = a_stream ? 1 : 0;

  CUtensorMap tmA, tmB;
  int st = make_map(&tmA, A, a_rows, kp, BM);
  if (st) return st;
  // gather mode: B is the whole operand table, rows picked by b_ids 4 at a time (box height 1)
  st = b_ids ? make_map(&tmB, B, b_table_rows, kp, 1) : make_map(&tmB, B, b_rows, kp, BN_HALF);
  if (st) return st;

  const size_t smem = smem_bytes(n_kb, stages, a_stream);
  static bool attr_set = false;
  if (!attr_set) {
    size_t mx = smem_bytes(5, 8);
    for (int kb = 6; kb <= kMaxKb; ++kb)
      if (smem_bytes(kb, 13 - kb) > mx) mx = smem_bytes(kb, 13 - kb);
    if (smem_bytes(0, kStreamStages, true) > mx) mx = smem_bytes(0, kStreamStages, true);
    cudaError_t e = cudaFuncSetAttribute(phase1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(phase1_kernel)");
    attr_set = true;
  }
  const int64_t n_units = (int64_t)((n_ranges + 1) / 2) * p.n_mpairs;
  const int64_t pairs = sm_count() / 2;
  const int grid = 2 * (int)(n_units < pairs ? n_units : pairs);
  ProfScope prof(stream, tag);
  phase1_kernel<<<grid, kThreads, smem, stream>>>(tmA, tmB, p);
  LCRW_CHECK_LAUNCH("phase1_kernel");
  return LCRW_OK;
}

}  // namespace p1
}  // namespace lcrw

#ifdef LCRW_P1_STATS
extern "C" int lcrw_p1_stats(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, lcrw::p1::g_p1_stats, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(lcrw::p1::g_p1_stats, z, sizeof(z));
  }
  return 0;
}
#endif

extern "C" int lcrw_phase1(const uint16_t* A, const float* a_norms, int64_t a_rows, const uint16_t* B,
                           int64_t b_rows, int m, int kp, const int64_t* seg_offsets,
                           int64_t seg_base, int64_t n_seg, const uint32_t* endmask, const int32_t* range_seg,
                           int64_t n_ranges, const float* scale, float* Z, int64_t z_panel, int z_shift,
                           void* stream) {
  return lcrw::p1::launch(A, a_norms, a_rows, B, b_rows, m, kp, seg_offsets, seg_base, n_seg, endmask,
                          range_seg, n_ranges, scale, Z, z_panel, z_shift, lcrw::as_stream(stream), "phase1");
}
