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
// Z holds (1 << zs)-segment panels (2 <= zs <= 7): with zs = 7 a warp's 128
// segments of one word row are one contiguous 512-byte run (four 128-byte
// lines per nonzero), with zs = 3 they are 16 separate 32-byte sectors.
// ---------------------------------------------------------------------------
// Z holding distances (finite, >= 0, zero or normal: the pipeline's Z1) lets the f32 -> f64
// widening run on the integer pipe: the f32 bits shifted into an f64 word are z * 2^-896
// exactly (exponent field kept, not rebiased; 0 stays 0), and the weight carries the 2^896,
// so fma(x * 2^896, z * 2^-896, acc) == fma(x, (double)z, acc) bit for bit, two shifts
// instead of an F2F on the XU pipe (16 lanes/clk/SM, which ncu shows saturated here).
__device__ __forceinline__ double dist_f64_scaled(float z) {
  const uint32_t b = __float_as_uint(z);
  return __hiloint2double((int)(b >> 3), (int)(b << 29));
}
#ifndef LCRW_SPMM_MINB
#define LCRW_SPMM_MINB 4  // 4 CTAs (32 warps) per SM, <= 64 registers: 8 row loads in flight per warp
                          // (C2: 16.6 ms; 5 CTAs / 48 registers 17.3 ms, unroll 16 at 80 registers 19.6 ms)
#endif
#ifndef LCRW_SPMM_UNROLL
#define LCRW_SPMM_UNROLL 8
#endif
constexpr int kSpmmUnroll = LCRW_SPMM_UNROLL;  // (#pragma unroll does not expand macros)
template <bool kDist>
__global__ void __launch_bounds__(kWarps * 32, LCRW_SPMM_MINB)
    spmm_kernel(const int64_t* __restrict__ offs, const int32_t* __restrict__ cols, const float* __restrict__ vals,
                int64_t n_rows, const float* __restrict__ Z, int64_t z_panel, int zs, int64_t z_block_rows,
                int64_t z_block_stride, int64_t n_seg, float* __restrict__ out, int64_t ld_row, int64_t ld_panel) {
  const int lane = threadIdx.x & 31;
  __shared__ longlong2 nz_s[kWarps][32];
  const int64_t q0 = (int64_t)blockIdx.y * kSegPerBlock + lane * 4;
  const bool active = q0 < n_seg;
  const float* zq = Z + (q0 >> zs) * z_panel + (q0 & ((1 << zs) - 1));
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
      const int64_t my_off = (int64_t)blk * z_block_stride + ((int64_t)(my_c - blk * zbr) << zs);
      // (offset, weight) of the 32 nonzeros staged per warp and read back as one broadcast
      // LDS.128 each, instead of three SHFLs (a 64-bit offset + the weight) that share the
      // L1TEX data pipe with the Z row loads
      // fast: distance Z and every weight of the block below 2^126 (always, for histogram
      // weights) -- the weights are staged pre-scaled by 2^896 (exact), one F2F per nonzero
      // instead of one per lane
      const bool fast = kDist && __all_sync(0xffffffffu, fabsf(my_x) < 0x1p126f);
      __syncwarp();
      nz_s[threadIdx.x >> 5][lane] =
          make_longlong2(my_off, __double_as_longlong(fast ? (double)my_x * 0x1p896 : (double)my_x));
      __syncwarp();
      int t0 = 0;
      // fast: a branch-free loop whose kSpmmUnroll row loads are all issued before the first
      // FMA (inactive lanes read segments 0-3 of the row -- panel 0, always allocated --
      // results unused), so each warp keeps kSpmmUnroll 512-byte runs in flight instead of
      // one; the FMAs run in the same ascending order, so the sums are bitwise those of the
      // loop below.
      if (fast) {
        const float* zl = active ? zq : Z;
        // (the block's last cnt % kSpmmUnroll nonzeros go through the loop below: a whole
        // last batch with weight-0 padding slots or predicated loads measured slower, and so
        // did loading the next block's ids ahead)
        for (; t0 + kSpmmUnroll <= cnt; t0 += kSpmmUnroll) {
          float4 z[kSpmmUnroll];
          double xs[kSpmmUnroll];
#pragma unroll
          for (int u = 0; u < kSpmmUnroll; ++u) {
            const longlong2 e = nz_s[threadIdx.x >> 5][t0 + u];
            z[u] = __ldg(reinterpret_cast<const float4*>(zl + e.x));  // (L1::no_allocate: 16.4 -> 23.8 ms)
            xs[u] = __longlong_as_double(e.y);
          }
#pragma unroll
          for (int u = 0; u < kSpmmUnroll; ++u) {
            a0 = fma(xs[u], dist_f64_scaled(z[u].x), a0);
            a1 = fma(xs[u], dist_f64_scaled(z[u].y), a1);
            a2 = fma(xs[u], dist_f64_scaled(z[u].z), a2);
            a3 = fma(xs[u], dist_f64_scaled(z[u].w), a3);
          }
        }
      }
      for (int t = t0; t < cnt; ++t) {
        const longlong2 e = nz_s[threadIdx.x >> 5][t];
        const int64_t zoff = e.x;
        const double x = __longlong_as_double(e.y);  // (pre-scaled by 2^896 when fast)
        if (active) {
          const float4 z = __ldg(reinterpret_cast<const float4*>(zq + zoff));
          if (fast || (kDist && fabs(x) < 0x1p126)) {  // (x * 2^896 stays finite; warp-uniform branch)
            const double xs = fast ? x : x * 0x1p896;
            a0 = fma(xs, dist_f64_scaled(z.x), a0);
            a1 = fma(xs, dist_f64_scaled(z.y), a1);
            a2 = fma(xs, dist_f64_scaled(z.z), a2);
            a3 = fma(xs, dist_f64_scaled(z.w), a3);
          } else {
            a0 = fma(x, (double)z.x, a0);
            a1 = fma(x, (double)z.y, a1);
            a2 = fma(x, (double)z.z, a2);
            a3 = fma(x, (double)z.w, a3);
          }
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
// Reverse direction, panel-streaming form.  Work item = (32-doc Z2 panel,
// group of <= 1024 queries); persistent CTAs (one per SM) loop over items.
// A producer warp streams each panel's word rows through a ring of 16 KB
// shared-memory tiles with 1-D TMA bulk copies -- each Z2 byte is read from
// HBM once (an L2 bulk prefetch running ahead of the ring measured slower:
// it competes with the ring's own bulk copies) -- and, into the same stage, the tile's block of the query plan (per-warp list
// ends + entries).  16 consumer warps scatter the entries, x * Z2[w, 32 docs],
// into per-query fp32 accumulators in shared memory.  Each query is owned by
// one warp ((q - q0) % 16), so its accumulation order is fixed by the plan:
// results are deterministic.  The plan packs every (tile, warp) list into
// groups of four entries of distinct queries, so a group's four accumulator
// read-modify-writes are independent and issue back to back.  The symmetric
// combine max(D1, D2) is written query-major (128-byte rows) for the
// per-query top-k.
// ---------------------------------------------------------------------------
constexpr int kRpWarps = 16;     // consumer warps (+1 producer warp)
constexpr int kRpTile = 128;     // Z2 rows per staged tile (16 KB)
constexpr int kRpStages = 5;
constexpr int kRpGroup = 1024;   // queries per work item
constexpr int kRpIlp = 4;        // entries per independent group (plan invariant)
constexpr int kRpBlkWords = 512;   // staged plan block per tile: 16 list ends + up to 248 entries (2 KB)
constexpr int kRpBlkEntries = (kRpBlkWords - kRpWarps) / 2;

// Fused max -> top-k of lcrw_reverse_panels: per (query, CTA slot) a sorted list of the k
// smallest (distance, id) seen so far, lists [q][slot][k] (d and i arrays), merged at the end
// by lcrw_topk_segments (kernels.py:210-232 order: ascending distance, then id).
struct TopLists {
  float* d;
  int64_t* i;
  int k;          // 1 .. 32
  int slots;      // list slots per query (>= grid)
  int64_t id_base;
};
constexpr float kInfF = __builtin_huge_valf();

// Inserts the candidates of ballot b (lane values v, ids id) into list `li` (entries
// li * k ..), held across lanes 0..k-1 while merging; returns the new k-th distance.
__device__ __forceinline__ float top_insert(const TopLists& t, int64_t li, uint32_t b, float v, int64_t id,
                                            int lane) {
  float* ld = t.d + li * t.k;
  int64_t* lid = t.i + li * t.k;
  const bool own = lane < t.k;
  float cur_d = own ? ld[lane] : kInfF;
  int64_t cur_i = own ? lid[lane] : INT64_MAX;
  while (b) {
    const int src = __ffs(b) - 1;
    b &= b - 1u;
    const float cd = __shfl_sync(0xffffffffu, v, src);
    const int64_t ci = __shfl_sync(0xffffffffu, id, src);
    // position = number of list entries ordered before the candidate
    const bool before = own && (cur_d < cd || (cur_d == cd && cur_i < ci));
    const int pos = __popc(__ballot_sync(0xffffffffu, before));
    const float up_d = __shfl_up_sync(0xffffffffu, cur_d, 1);
    const int64_t up_i = __shfl_up_sync(0xffffffffu, cur_i, 1);
    if (pos < t.k && lane >= pos) {
      cur_d = lane == pos ? cd : up_d;
      cur_i = lane == pos ? ci : up_i;
    }
  }
  if (own) {
    ld[lane] = cur_d;
    lid[lane] = cur_i;
  }
  return __shfl_sync(0xffffffffu, cur_d, t.k - 1);
}

__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

__global__ void __launch_bounds__((kRpWarps + 1) * 32, 1)
    reverse_panels_kernel(const float* __restrict__ Z2, int64_t z_panel, int64_t a_rows, int64_t n_docs,
                          int64_t doc_base, const uint32_t* __restrict__ e_blk, const int64_t* __restrict__ e_tile,
                          int n_tiles, int64_t n_q, const float* __restrict__ D1, int64_t d1_ld_panel,
                          float* __restrict__ D, int64_t ld_q, int64_t ld_doc, int64_t n_panels, int64_t n_items,
                          TopLists top) {
  extern __shared__ __align__(16) float rp_smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  float* acc = rp_smem;            // [kRpGroup + kRpWarps][32] (+ one scratch row per warp for padding entries)
  float* tiles = acc + (kRpGroup + kRpWarps) * 32;                              // [kRpStages][kRpTile][32]
  uint32_t* blks = reinterpret_cast<uint32_t*>(tiles + kRpStages * kRpTile * 32);  // [kRpStages][kRpBlkWords]
  uint64_t* full = reinterpret_cast<uint64_t*>(blks + kRpStages * kRpBlkWords);
  uint64_t* empty = full + kRpStages;
  float* thr = reinterpret_cast<float*>(empty + kRpStages);  // [kRpGroup] top-k mode: k-th distance per query
  for (int i = threadIdx.x; i < (kRpGroup + kRpWarps) * 32; i += blockDim.x) acc[i] = 0.f;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kRpStages; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, kRpWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kRpWarps) {
    // ---- producer warp: lane 0 issues, the lanes fetch plan offsets 32 tiles at a time ----
    uint32_t it = 0;
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int64_t p = item % n_panels;
      const int64_t g = item / n_panels;
      const float* zp = Z2 + p * z_panel;
      const int64_t* tb = e_tile + g * n_tiles;
      // D1 lines of this item, needed by the consumers' combine at the end
      {
        const int64_t q0 = g * kRpGroup;
        const int nqp = (int)((min((int64_t)kRpGroup, n_q - q0) + 7) / 8);
        const int64_t j0 = doc_base + p * 32;
        const uint32_t dbytes = (uint32_t)min((int64_t)32, n_docs - p * 32) * 32u;
        for (int qp = lane; qp < nqp; qp += 32) bulk_prefetch_l2(D1 + ((q0 >> 3) + qp) * d1_ld_panel + j0 * 8, dbytes);
      }
      int64_t b_lo = 0, b_hi = 0;
      for (int t = 0; t < n_tiles; ++t, ++it) {
        if ((t & 31) == 0) {  // plan block offsets of tiles t .. t+32
          const int n = min(33, n_tiles + 1 - t);
          b_lo = lane < n ? __ldg(tb + t + lane) : 0;
          b_hi = lane == 0 && n == 33 ? __ldg(tb + t + 32) : 0;  // the 33rd offset
        }
        const int64_t blk0 = __shfl_sync(0xffffffffu, b_lo, t & 31);
        const int64_t blk1 = (t & 31) == 31 ? __shfl_sync(0xffffffffu, b_hi, 0)
                                            : __shfl_sync(0xffffffffu, b_lo, (t & 31) + 1);
        const uint32_t st = it % kRpStages;
        mbar_wait(empty + st, ((it / kRpStages) & 1) ^ 1);
        if (lane == 0) {
          const int64_t r0 = (int64_t)t * kRpTile;
          const uint32_t zbytes = (uint32_t)min((int64_t)kRpTile, a_rows - r0) * 128u;
          const uint32_t bbytes = (uint32_t)min((int64_t)kRpBlkWords, blk1 - blk0) * 4u;
          mbar_expect_tx(full + st, zbytes + bbytes);
          bulk_load(tiles + st * kRpTile * 32, zp + r0 * 32, zbytes, full + st);
          bulk_load(blks + st * kRpBlkWords, e_blk + blk0, bbytes, full + st);
        }
        __syncwarp();
      }
    }
    return;
  }

  // ---- consumers ----
  // stage / phase tracked incrementally (no div/mod by kRpStages per tile)
  uint32_t st = 0, ph = 0;
  int64_t top_g = -1;  // query group whose thresholds are in thr
  const char* acc_lane = reinterpret_cast<const char*>(acc + lane);
  for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int64_t p = item % n_panels;
    const int64_t g = item / n_panels;
    const int64_t q0 = g * kRpGroup;
    const int nq = (int)min((int64_t)kRpGroup, n_q - q0);
    for (int t = 0; t < n_tiles; ++t) {
      mbar_wait(full + st, ph);
      const char* tile_lane = reinterpret_cast<const char*>(tiles + st * (kRpTile * 32) + lane);
      const uint32_t* blk = blks + st * kRpBlkWords;
      const int e0 = warp ? (int)blk[warp - 1] : 0;
      const int e1 = (int)blk[warp];
      // entry word: (row * 128) << 18 | query * 128 -- byte offsets of the tile row and accumulator row
      auto scatter = [&](uint4 ab, uint4 cd) {
        const uint32_t pk[kRpIlp] = {ab.x, ab.z, cd.x, cd.z};
        const float x[kRpIlp] = {__uint_as_float(ab.y), __uint_as_float(ab.w), __uint_as_float(cd.y),
                                 __uint_as_float(cd.w)};
        float* a[kRpIlp];
        float z[kRpIlp], v[kRpIlp];
#pragma unroll
        for (int j = 0; j < kRpIlp; ++j) {
          a[j] = reinterpret_cast<float*>(const_cast<char*>(acc_lane) + (pk[j] & 0x3FFFFu));
          z[j] = *reinterpret_cast<const float*>(tile_lane + (pk[j] >> 18));
          v[j] = *a[j];
        }
#pragma unroll
        for (int j = 0; j < kRpIlp; ++j) *a[j] = fmaf(x[j], z[j], v[j]);
      };
      constexpr int kStaged = kRpBlkEntries / kRpIlp * kRpIlp;
      const int e_mid = e1 < kStaged ? e1 : kStaged;
      const uint4* ep = reinterpret_cast<const uint4*>(blk + kRpWarps) + (e0 >> 1);
      for (int i = e0; i < e_mid; i += kRpIlp, ep += 2) scatter(ep[0], ep[1]);
      if (e1 > kStaged) {  // rare: the tile's plan block exceeds the staged part; the rest comes from global
        const uint4* gent = reinterpret_cast<const uint4*>(e_blk + __ldg(e_tile + g * n_tiles + t) + kRpWarps);
        for (int i = e0 > kStaged ? e0 : kStaged; i < e1; i += kRpIlp) scatter(__ldg(gent + (i >> 1)), __ldg(gent + (i >> 1) + 1));
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + st);
      if (++st == kRpStages) {
        st = 0;
        ph ^= 1;
      }
    }
    named_bar_sync(1, kRpWarps * 32);  // all scatters of this item are in acc

    // symmetric combine with D1 (8-query panels: D1[(q >> 3) * ld_panel + j * 8 + (q & 7)]); re-zero acc
    const int64_t j = p * 32 + lane;
    const bool valid = j < n_docs;
    const int64_t jg = doc_base + j;
    if (top.d) {
      // fused max -> top-k (no D): this CTA's running k best per query (its list slot), the
      // k-th distance cached in smem; a warp owns its queries, so no two warps touch a list
      if (g != top_g) {
        for (int ql = warp * 32 + lane; ql < nq; ql += kRpWarps * 32)
          thr[ql] = top.d[((q0 + ql) * top.slots + blockIdx.x) * top.k + top.k - 1];
        top_g = g;
        named_bar_sync(1, kRpWarps * 32);
      }
      for (int qp = warp; qp * 8 < nq; qp += kRpWarps) {
        const int64_t qg = q0 + qp * 8;
        float d1v[8];
        if (valid) {
          const float4* src = reinterpret_cast<const float4*>(D1 + (qg >> 3) * d1_ld_panel + jg * 8);
          const float4 lo4 = __ldg(src), hi4 = __ldg(src + 1);
          d1v[0] = lo4.x; d1v[1] = lo4.y; d1v[2] = lo4.z; d1v[3] = lo4.w;
          d1v[4] = hi4.x; d1v[5] = hi4.y; d1v[6] = hi4.z; d1v[7] = hi4.w;
        }
#pragma unroll
        for (int qq = 0; qq < 8; ++qq) {
          const int ql = qp * 8 + qq;
          if (ql < nq) {
            float* a = acc + ql * 32 + lane;
            const float v = valid ? fmaxf(d1v[qq], *a) : kInfF;
            *a = 0.f;
            const uint32_t b = __ballot_sync(0xffffffffu, valid && v <= thr[ql]);
            if (b) {
              const float kth = top_insert(top, (q0 + ql) * top.slots + blockIdx.x, b, v, jg + top.id_base, lane);
              __syncwarp();  // every lane's read of thr[ql] precedes the update
              if (lane == 0) thr[ql] = kth;
              __syncwarp();
            }
          }
        }
      }
      named_bar_sync(1, kRpWarps * 32);  // acc is zero again before the next item's scatter
      continue;
    }
    for (int qp = warp; qp * 8 < nq; qp += kRpWarps) {
      const int64_t qg = q0 + qp * 8;
      float d1v[8];
      if (valid) {
        const float4* src = reinterpret_cast<const float4*>(D1 + (qg >> 3) * d1_ld_panel + jg * 8);
        const float4 lo4 = __ldg(src), hi4 = __ldg(src + 1);
        d1v[0] = lo4.x; d1v[1] = lo4.y; d1v[2] = lo4.z; d1v[3] = lo4.w;
        d1v[4] = hi4.x; d1v[5] = hi4.y; d1v[6] = hi4.z; d1v[7] = hi4.w;
      }
#pragma unroll
      for (int qq = 0; qq < 8; ++qq) {
        const int ql = qp * 8 + qq;
        if (ql < nq) {
          float* a = acc + ql * 32 + lane;
          if (valid) D[(qg + qq) * ld_q + jg * ld_doc] = fmaxf(d1v[qq], *a);
          *a = 0.f;
        }
      }
    }
    named_bar_sync(1, kRpWarps * 32);  // acc is zero again before the next item's scatter
  }
}



// ---------------------------------------------------------------------------
// All-pairs symmetric combine (X1 == X2): the reverse direction of a pair is the
// forward direction of the swapped pair, so D = max(D1, D1^T) in place.  One
// 32x32 tile pair per CTA (upper-triangle tiles only), transposed through
// shared memory so both reads and both writes are coalesced.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) symmetrize_max_kernel(float* __restrict__ D, int64_t n, int64_t ld) {
  __shared__ float ta[32][33], tb[32][33];
  const int64_t bi = blockIdx.y, bj = blockIdx.x;
  if (bj < bi) return;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
  const int64_t r0 = bi * 32, c0 = bj * 32;
  for (int y = ty; y < 32; y += 8) {
    const int64_t r = r0 + y, c = c0 + tx;
    ta[y][tx] = (r < n && c < n) ? D[r * ld + c] : 0.f;      // tile (bi, bj)
    const int64_t r2 = c0 + y, c2 = r0 + tx;
    tb[y][tx] = (r2 < n && c2 < n) ? D[r2 * ld + c2] : 0.f;  // tile (bj, bi)
  }
  __syncthreads();
  for (int y = ty; y < 32; y += 8) {
    const int64_t r = r0 + y, c = c0 + tx;
    if (r < n && c < n) D[r * ld + c] = fmaxf(ta[y][tx], tb[tx][y]);
    const int64_t r2 = c0 + y, c2 = r0 + tx;
    if (r2 < n && c2 < n) D[r2 * ld + c2] = fmaxf(tb[y][tx], ta[tx][y]);
  }
}


// out[i, j] = max(A[i, j], R[j, i]) for i < rows, j < cols: the sharded all-pairs combine
// (a peer's block of the forward bounds against this rank's own block, transposed through
// smem).  out may alias A (the in-place lcrw_max_transposed).
__global__ void __launch_bounds__(256) max_transposed_kernel(float* out, int64_t ldo, const float* A, int64_t lda,
                                                             const float* __restrict__ R, int64_t ldr, int64_t rows,
                                                             int64_t cols) {
  __shared__ float t[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t i0 = (int64_t)blockIdx.y * 32, j0 = (int64_t)blockIdx.x * 32;
  for (int y = ty; y < 32; y += 8) {  // R rows j0 + y, columns i0 + tx
    const int64_t j = j0 + y, i = i0 + tx;
    t[y][tx] = (j < cols && i < rows) ? R[j * ldr + i] : 0.f;
  }
  __syncthreads();
  for (int y = ty; y < 32; y += 8) {
    const int64_t i = i0 + y, j = j0 + tx;
    if (i < rows && j < cols) out[i * ldo + j] = fmaxf(A[i * lda + j], t[tx][y]);
  }
}

}  // namespace p2
}  // namespace lcrw

using namespace lcrw;
using namespace lcrw::p2;

extern "C" {

static int spmm_launch(bool dist, const int64_t* offs, const int32_t* cols, const float* vals, int64_t n_rows,
                       const float* Z, int64_t z_panel, int z_shift, int64_t z_block_rows, int64_t z_block_stride,
                       int64_t n_seg, float* out, int64_t ld_row, int64_t ld_panel, void* stream) {
  LCRW_REQUIRE(n_rows >= 0 && n_seg >= 0, "lcrw_spmm: bad shape");
  if (n_rows == 0 || n_seg == 0) return LCRW_OK;
  LCRW_REQUIRE(offs && cols && vals && Z && out, "lcrw_spmm: null pointer");
  LCRW_REQUIRE(z_shift >= 2 && z_shift <= 7, "lcrw_spmm: z_shift must be in [2, 7]");
  LCRW_REQUIRE(z_panel % 4 == 0 && z_block_stride % 4 == 0 && (reinterpret_cast<uintptr_t>(Z) & 15) == 0,
               "lcrw_spmm: Z must be 16-byte aligned with z_panel, z_block_stride % 4 == 0");
  if (z_block_rows <= 0) z_block_rows = INT64_MAX;
  const int64_t gy = ceil_div(n_seg, kSegPerBlock);
  LCRW_REQUIRE(gy < 65536, "lcrw_spmm: too many segments for one launch");
  int64_t gx = ceil_div(n_rows, kWarps);
  const int64_t cap = (int64_t)sm_count() * 64;
  if (gx > cap) gx = cap;
  ProfScope prof(as_stream(stream), "spmm");
  const dim3 grid((unsigned)gx, (unsigned)gy);
  if (dist)
    spmm_kernel<true><<<grid, kWarps * 32, 0, as_stream(stream)>>>(offs, cols, vals, n_rows, Z, z_panel, z_shift,
                                                                  z_block_rows, z_block_stride, n_seg, out, ld_row,
                                                                  ld_panel);
  else
    spmm_kernel<false><<<grid, kWarps * 32, 0, as_stream(stream)>>>(offs, cols, vals, n_rows, Z, z_panel, z_shift,
                                                                   z_block_rows, z_block_stride, n_seg, out, ld_row,
                                                                   ld_panel);
  LCRW_CHECK_LAUNCH("spmm_kernel");
  return LCRW_OK;
}

int lcrw_spmm(const int64_t* offs, const int32_t* cols, const float* vals, int64_t n_rows, const float* Z,
              int64_t z_panel, int z_shift, int64_t z_block_rows, int64_t z_block_stride, int64_t n_seg, float* out,
              int64_t ld_row, int64_t ld_panel, void* stream) {
  return spmm_launch(false, offs, cols, vals, n_rows, Z, z_panel, z_shift, z_block_rows, z_block_stride, n_seg, out,
                     ld_row, ld_panel, stream);
}

int lcrw_spmm_dist(const int64_t* offs, const int32_t* cols, const float* vals, int64_t n_rows, const float* Z,
                   int64_t z_panel, int z_shift, int64_t z_block_rows, int64_t z_block_stride, int64_t n_seg,
                   float* out, int64_t ld_row, int64_t ld_panel, void* stream) {
  return spmm_launch(true, offs, cols, vals, n_rows, Z, z_panel, z_shift, z_block_rows, z_block_stride, n_seg, out,
                     ld_row, ld_panel, stream);
}


int lcrw_symmetrize_max(float* D, int64_t n, int64_t ld, void* stream) {
  LCRW_REQUIRE(n >= 0 && ld >= n, "lcrw_symmetrize_max: bad shape");
  if (n == 0) return LCRW_OK;
  LCRW_REQUIRE(D, "lcrw_symmetrize_max: null pointer");
  const int64_t t = ceil_div(n, 32);
  LCRW_REQUIRE(t < 65536, "lcrw_symmetrize_max: n too large for one launch");
  cudaStream_t st = as_stream(stream);
  ProfScope prof(st, "symmetrize");
  symmetrize_max_kernel<<<dim3((unsigned)t, (unsigned)t), 256, 0, st>>>(D, n, ld);
  LCRW_CHECK_LAUNCH("symmetrize_max_kernel");
  return LCRW_OK;
}

int lcrw_max_transposed_into(float* out, int64_t ldo, const float* A, int64_t lda, const float* R, int64_t ldr,
                             int64_t rows, int64_t cols, void* stream) {
  LCRW_REQUIRE(rows >= 0 && cols >= 0 && ldo >= cols && lda >= cols && ldr >= rows,
               "lcrw_max_transposed: bad shape");
  if (rows == 0 || cols == 0) return LCRW_OK;
  LCRW_REQUIRE(out && A && R, "lcrw_max_transposed: null pointer");
  LCRW_REQUIRE(ceil_div(rows, 32) < 65536, "lcrw_max_transposed: too many rows for one launch");
  cudaStream_t st = as_stream(stream);
  max_transposed_kernel<<<dim3((unsigned)ceil_div(cols, 32), (unsigned)ceil_div(rows, 32)), 256, 0, st>>>(
      out, ldo, A, lda, R, ldr, rows, cols);
  LCRW_CHECK_LAUNCH("max_transposed_kernel");
  return LCRW_OK;
}

int lcrw_max_transposed(float* D, int64_t ldd, const float* R, int64_t ldr, int64_t rows, int64_t cols,
                        void* stream) {
  return lcrw_max_transposed_into(D, ldd, D, ldd, R, ldr, rows, cols, stream);
}

int lcrw_reverse_panels_tile_rows(void) { return kRpTile; }
int lcrw_reverse_panels_group(void) { return kRpGroup; }
int lcrw_reverse_panels_warps(void) { return kRpWarps; }
int lcrw_reverse_panels_ilp(void) { return kRpIlp; }

int lcrw_reverse_panels_top_slots(void) { return sm_count(); }

int lcrw_reverse_panels(const float* Z2, int64_t z_panel, int64_t a_rows, int64_t n_docs, int64_t doc_base,
                        const uint32_t* e_blk, const int64_t* e_tile, int64_t n_q, const float* D1,
                        int64_t d1_ld_panel, float* D, int64_t ld_q, int64_t ld_doc, float* top_d, int64_t* top_i,
                        int k, int64_t id_base, void* stream) {
  LCRW_REQUIRE(n_q >= 0 && n_docs >= 0 && a_rows >= 0, "lcrw_reverse_panels: bad shape");
  if (n_q == 0 || n_docs == 0) return LCRW_OK;
  LCRW_REQUIRE(Z2 && e_blk && e_tile && D1 && (D || top_d), "lcrw_reverse_panels: null pointer");
  LCRW_REQUIRE(!top_d || (top_i && k >= 1 && k <= 32), "lcrw_reverse_panels: top-k lists need ids and 1 <= k <= 32");
  LCRW_REQUIRE(z_panel == a_rows * 32 && (reinterpret_cast<uintptr_t>(Z2) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(e_blk) & 15) == 0 && (reinterpret_cast<uintptr_t>(D1) & 15) == 0,
               "lcrw_reverse_panels: Z2 (32-doc panels, z_panel = 32 * a_rows), e_blk and D1 must be 16-byte aligned");
  const int64_t n_tiles = ceil_div(a_rows, kRpTile);
  const int64_t panels = ceil_div(n_docs, 32);
  const int64_t groups = ceil_div(n_q, kRpGroup);
  LCRW_REQUIRE(n_tiles < (1 << 30), "lcrw_reverse_panels: query vocabulary too large");
  const int smem = ((kRpGroup + kRpWarps) * 32 + kRpStages * kRpTile * 32 + kRpStages * kRpBlkWords) * 4 +
                   2 * kRpStages * 8 + kRpGroup * 4;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(reverse_panels_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(reverse_panels_kernel)");
    attr = true;
  }
  const int64_t items = panels * groups;
  const int64_t grid = items < sm_count() ? items : sm_count();
  cudaStream_t st = as_stream(stream);
  ProfScope prof(st, "reverse_panels");
  reverse_panels_kernel<<<(unsigned)grid, (kRpWarps + 1) * 32, smem, st>>>(
      Z2, z_panel, a_rows, n_docs, doc_base, e_blk, e_tile, (int)n_tiles, n_q, D1, d1_ld_panel, D, ld_q, ld_doc,
      panels, items, TopLists{top_d, top_i, k, sm_count(), id_base});
  LCRW_CHECK_LAUNCH("reverse_panels_kernel");
  return LCRW_OK;
}

}  // extern "C"
