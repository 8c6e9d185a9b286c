// Shared device helpers for the LC-RWMD sm_100a kernels: inline-PTX wrappers
// for mbarriers, TMA, tcgen05 (MMA / TMEM) and the thread-local error slot
// behind the C ABI.
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/lcrwmd.h"

namespace lcrw {

// ---------------------------------------------------------------------------
// host-side error plumbing (abi.cu)
// ---------------------------------------------------------------------------
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* what);

#define LCRW_CHECK_LAUNCH(what)                                   \
  do {                                                            \
    cudaError_t e_ = cudaGetLastError();                          \
    if (e_ != cudaSuccess) return ::lcrw::cuda_status(e_, what);  \
  } while (0)

#define LCRW_REQUIRE(cond, msg)                  \
  do {                                           \
    if (!(cond)) {                               \
      ::lcrw::set_error("%s", msg);              \
      return LCRW_ERR_INVALID;                   \
    }                                            \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// RAII event pair around a launch when the profiler is enabled (abi.cu)
class ProfScope {
 public:
  ProfScope(cudaStream_t s, const char* name);
  ~ProfScope();
  ProfScope(const ProfScope&) = delete;
  ProfScope& operator=(const ProfScope&) = delete;

 private:
  cudaStream_t stream_;
  const char* name_;
  cudaEvent_t a_;
};
int sm_count();
int64_t ceil_div(int64_t a, int64_t b);

// ---------------------------------------------------------------------------
// device: shared-memory addressing, mbarriers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!done);
}

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------------------
// TMA (cp.async.bulk.tensor) -- 2-D tile loads completing on an mbarrier
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}

__device__ __forceinline__ void tma_load_2d(const CUtensorMap* m, uint64_t* bar, void* dst, int32_t c0,
                                            int32_t c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}

// 1-D bulk copy global -> shared (16-byte aligned, size multiple of 16) completing on an mbarrier
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// ---------------------------------------------------------------------------
// clusters (CTA pairs)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same smem variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_shared(uint32_t local_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(rank));
  return r;
}
// relaxed: orders nothing but the arrival itself (TMEM reads are ordered by
// tcgen05.fence::before_thread_sync; global stores need no ordering here)
__device__ __forceinline__ void mbar_arrive_cluster_relaxed(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// 2-SM TMA: data lands in this CTA's smem, completion bytes go to the barrier at
// the given shared::cluster address (the leader CTA's barrier).
__device__ __forceinline__ void tma_load_2d_2sm(const CUtensorMap* m, uint32_t bar_cluster_addr, void* dst,
                                                int32_t c0, int32_t c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_cluster_addr), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}

// 2-SM TMA gather: 4 rows (row indices r0..r3) x one box of columns starting at c0 land as
// 4 consecutive rows at dst in this CTA's smem (swizzled by address like a tile load);
// completion bytes go to the barrier at the given shared::cluster address.
__device__ __forceinline__ void tma_gather4_2sm(const CUtensorMap* m, uint32_t bar_cluster_addr, void* dst,
                                                int32_t c0, int32_t r0, int32_t r1, int32_t r2, int32_t r3,
                                                uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%3, %4, %5, %6, %7}], [%2], %8;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_cluster_addr), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
      "l"(policy)
      : "memory");
}

// ---------------------------------------------------------------------------
// tcgen05: TMEM allocation, UMMA issue/commit, TMEM -> register loads
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc_2sm(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tmem_relinquish_2sm() {
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_2sm(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
// pair MMA issued by the leader CTA: A rows split across the two CTAs (M = 256),
// B columns split across the two CTAs' smem (N/2 each), D in each CTA's TMEM.
__device__ __forceinline__ void umma_f16_2sm(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// warp-wide variants: every lane executes with warp-uniform operands and one
// elected lane issues, so the compiler keeps descriptors in uniform registers
__device__ __forceinline__ void umma_f16_2sm_elect(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                   uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit_2sm_mc_elect(uint64_t* bar, uint16_t cta_mask) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}"
      ::"r"(smem_u32(bar)), "h"(cta_mask)
      : "memory");
}
// arrive (once) on the barrier at the same smem offset in every CTA of cta_mask
__device__ __forceinline__ void umma_commit_2sm_mc(uint64_t* bar, uint16_t cta_mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(cta_mask)
      : "memory");
}

__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tmem_relinquish() {
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// K-major operand tile in the canonical 128-byte-swizzle layout written by
// TMA (rows of 128 B, 8-row groups 1024 B apart): LBO = 16 B (unused for
// swizzled K-major), SBO = 1024 B, version 1 (sm_100), layout SWIZZLE_128B.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  return static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) |
         (static_cast<uint64_t>(2) << 61);
}

// kind::f16 instruction descriptor: A,B f16 K-major, D f32, shape M x N.
__host__ __device__ constexpr uint32_t umma_idesc_f16(int M, int N) {
  return (1u << 4) | (0u << 7) | (0u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// 32 lanes x 32 consecutive 32-bit columns: thread t gets row (lane base + t).
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
        "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
        "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
        "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr)
      : "memory");
}

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ---------------------------------------------------------------------------
// ordering helpers
// ---------------------------------------------------------------------------
// Monotone map float -> uint32 (total order for non-NaN values).
// order-preserving unsigned key of a float under numpy's sort order: -0 == +0, and every
// NaN after +inf (one key for all NaNs, so NaNs tie and fall back to the id)
__device__ __forceinline__ uint32_t float_key(float d) {
  uint32_t u = __float_as_uint(d);
  if ((u & 0x7FFFFFFFu) > 0x7F800000u) return 0xFFFFFFFFu;
  if (u == 0x80000000u) u = 0u;
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key_float(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}

// ---------------------------------------------------------------------------
// 16-bit distance keys of the reverse direction (table.cu).
// Reverse-direction distances are stored as 16-bit keys relative to their query-
// vocabulary word w (the table's column; the A row of the Phase-1 GEMM): with |w|^2 the
// A row's scaled squared norm and 2^e <= |w| / 2 < 2^(e+1) (key16_base),
//   0          exact zero (identical rows);
//   1          0 < d < 2^e (below the range: a near entry, d < |w| / 2, refined exactly;
//              decodes to 2^(e-1));
//   2..0xFFFE  d in [2^e, 2^(e+4)): 2 exponent bits (the binade above 2^e) and 14 mantissa
//              bits, rounded to nearest (relative error <= 2^-15 ~ 3.1e-5);
//   0xFFFF     saturated: d at or above the top of the range (> 4 |w|), refined exactly.
// Codes of one word compare like its distances, so a doc's minimum over its words' rows
// is an integer minimum, and the table form and the GEMM form of the reverse Phase 1
// (which rounds its Z2 through the same key) give identical Z2.
// ---------------------------------------------------------------------------
constexpr uint32_t kKey16Sat = 0xFFFFu;
__device__ __forceinline__ uint32_t key16_base(float a_sq) {  // bits of 2^e (f32)
  const int e2 = (int)(__float_as_uint(a_sq) >> 23) - 127;   // exponent of |w|^2
  return (uint32_t)((e2 >> 1) - 1 + 127) << 23;               // 2^e <= |w| / 2 < 2^(e+1)
}
// (branch-free: selects, so an epilogue's independent encodes interleave)
__device__ __forceinline__ uint32_t dist_key16(float d, uint32_t base) {
  const uint32_t b = __float_as_uint(d);
  uint32_t c = min(max((b - base + 256u) >> 9, 1u), kKey16Sat);
  c = b < base ? 1u : c;
  return b == 0u ? 0u : c;
}
__device__ __forceinline__ float key16_dist(uint32_t c, uint32_t base) {
  const uint32_t bits = c == 1u ? base - (1u << 23) : base + (c << 9);
  return c == 0u ? 0.f : __uint_as_float(bits);
}
// the decoded value of a saturated key: an entry at it is refined exactly
__device__ __forceinline__ float key16_sat(uint32_t base) { return key16_dist(kKey16Sat, base); }
// Near-entry refinement (refine.cu): a Z entry whose scaled distance d satisfies
// 0 < d < kRefineTau * |a| (|a|^2 = the A row's scaled squared norm) is recomputed
// exactly from the f32 rows.  The test always reads the stored (unscaled) Z value times
// the power-of-two scale, so table_min's list and the GEMM form's scan of the same Z2
// flag the same entries.
constexpr float kRefineTau = 0.5f;
__device__ __forceinline__ bool refine_flag(float d_scaled, float a_sq, float tau2) {
  return d_scaled > 0.f && d_scaled * d_scaled < tau2 * a_sq;
}
// where a reverse-pass producer appends the (row, segment) pairs it flags (64-bit count:
// a heavily clustered batch can flag more than 2^32 entries)
struct RefineSink {
  uint2* list;
  unsigned long long* count;
  int64_t cap;
};
// Marked entries (near pairs, near.cu): a producer that flags an entry stores kZMarked
// (all bits set) instead of its value; lcrw_near_scatter lowers a marked entry with
// atomicMin(kZMarkBit | bits(exact distance)) -- unmarked entries are non-negative floats,
// below kZMarkBit, and never change -- and lcrw_refine_near's finalize mode clears the
// mark bit, or recomputes an entry no near pair reached (still kZMarked).
constexpr uint32_t kZMarkBit = 0x80000000u;
constexpr uint32_t kZMarked = 0xFFFFFFFFu;
// near pairs (near.cu): candidates are the word pairs whose table distance is below
// kNearCandTau * max(|a|, |b|) (+ an absolute f16-subnormal term); kept as near pairs of a
// direction when the exact distance is below kNearTau * |row word| -- a margin of 0.15 max
// norm over the Gram error and of 0.1 |a| over the refine test
constexpr float kNearTau = 0.6f;
constexpr float kNearCandTau = 0.75f;
// exact squared distance sum_k (a_k - b_k)^2 of two f32 rows, warp-cooperative (lanes
// split the m dimensions, xor-reduction; every lane returns it).  The one formula of every
// exact re-evaluation (refine.cu, near.cu): (a - b)^2 == (b - a)^2 bitwise, so a pair gives
// the same value in either role.
__device__ __forceinline__ float exact_sq(const float* __restrict__ a, const float* __restrict__ b, int m,
                                          int lane) {
  float acc = 0.f;
  for (int k = lane; k < m; k += 32) {
    const float diff = __ldg(a + k) - __ldg(b + k);
    acc = fmaf(diff, diff, acc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}
// Table rows: 256 query-vocabulary words per chunk; per vocabulary word u one 512-byte
// row of 256 little-endian 16-bit keys (word w of the chunk at byte 2 w): 32 16-byte groups
// of 8 keys, one per lane in table_min (2 bytes per distance; the minima are SIMD 16-bit
// integer minima, VIMNMX.U16x2).  The table build (phase1 epilogue, kZTable) stores a
// warp's 32 rows (= 32 consecutive words) of one column as 64 contiguous bytes.
constexpr int kTableChunk = 256;
constexpr int kTableKeysPerGroup = 8;
constexpr int kTableGroups = 32;
constexpr int kTableRowBytes = 512;

namespace p1 {
// the tcgen05 Phase-1 GEMM with fused segmented-min epilogue (phase1.cu)
int launch(const uint16_t* A, const float* a_norms, int64_t a_rows, const uint16_t* B, int64_t b_rows, int m, int kp,
           const int64_t* seg_offsets, int64_t seg_base, int64_t n_seg, const uint32_t* endmask,
           const int32_t* range_seg, int64_t n_ranges, const float* scale, float* Z, int64_t z_panel, int z_shift,
           cudaStream_t stream, const char* tag, const int32_t* b_ids = nullptr, int64_t b_table_rows = 0,
           int z_mode = 0);
}  // namespace p1

}  // namespace lcrw
