// Top-k selection under ascending (distance, id) (kernels.py:210-232).
//
// lcrw_topk_segments: one CTA per segment keeps the current best KP (power of
// two >= k) entries sorted at the front of a 2048-entry shared buffer;
// candidates that beat the running k-th entry are appended and the buffer is
// re-sorted with a bitonic network only when something was appended.  The
// filter is exact (an entry not better than the k-th can never enter), so the
// result equals a full lexicographic sort truncated to k.
#include <cub/cub.cuh>

#include "common.cuh"

namespace lcrw {
namespace tk {

constexpr int kBuf = 2048;
constexpr int kThreads = 1024;

struct Entry {
  uint32_t key;  // float_key(distance)
  int64_t id;
};

__device__ __forceinline__ bool less(uint32_t ka, int64_t ia, uint32_t kb, int64_t ib) {
  return ka < kb || (ka == kb && ia < ib);
}

__device__ void bitonic_sort(uint32_t* key, int64_t* id) {
  for (int size = 2; size <= kBuf; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int t = threadIdx.x; t < kBuf / 2; t += blockDim.x) {
        const int i = 2 * t - (t & (stride - 1));
        const int j = i + stride;
        const bool up = ((i & size) == 0);
        const uint32_t ki = key[i], kj = key[j];
        const int64_t ii = id[i], ij = id[j];
        const bool swap = up ? less(kj, ij, ki, ii) : less(ki, ii, kj, ij);
        if (swap) {
          key[i] = kj;
          key[j] = ki;
          id[i] = ij;
          id[j] = ii;
        }
      }
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kThreads)
    topk_segments_kernel(const float* __restrict__ d, const int64_t* __restrict__ ids, int64_t ld, int64_t seg_len,
                         int64_t id_base, int k, int kp, float* __restrict__ out_d, int64_t* __restrict__ out_i) {
  __shared__ uint32_t key[kBuf];
  __shared__ int64_t idb[kBuf];
  __shared__ int count;
  const int64_t seg = blockIdx.x;
  // ids == NULL: implicit ids id_base + position (rows of a distance matrix)
  const float* ds = d + seg * ld;
  const int64_t* is = ids ? ids + seg * ld : nullptr;
  for (int i = threadIdx.x; i < kBuf; i += blockDim.x) {
    key[i] = 0xFFFFFFFFu;
    idb[i] = INT64_MAX;
  }
  if (threadIdx.x == 0) count = 0;
  __syncthreads();
  const int cap = kBuf - kp;  // append area (>= 1024 == blockDim)
  for (int64_t base = 0; base < seg_len; base += blockDim.x) {
    const uint32_t thr_k = key[k - 1];
    const int64_t thr_i = idb[k - 1];
    const int64_t i = base + threadIdx.x;
    if (i < seg_len) {
      const uint32_t kk = float_key(ds[i]);
      const int64_t ii = is ? is[i] : id_base + i;
      if (less(kk, ii, thr_k, thr_i)) {
        const int pos = atomicAdd(&count, 1);
        key[kp + pos] = kk;
        idb[kp + pos] = ii;
      }
    }
    __syncthreads();
    const int n_new = count;
    if (n_new > 0) {
      for (int t = kp + n_new + threadIdx.x; t < kBuf; t += blockDim.x) {
        key[t] = 0xFFFFFFFFu;
        idb[t] = INT64_MAX;
      }
      bitonic_sort(key, idb);
      if (threadIdx.x == 0) count = 0;
      // the tail beyond kp is garbage-free after the sort (sentinels refilled next round)
      for (int t = kp + threadIdx.x; t < kBuf; t += blockDim.x) {
        key[t] = 0xFFFFFFFFu;
        idb[t] = INT64_MAX;
      }
    }
    __syncthreads();
    (void)cap;
  }
  const int kk = (int)min((int64_t)k, seg_len);
  for (int r = threadIdx.x; r < kk; r += blockDim.x) {
    out_d[seg * k + r] = key_float(key[r]);
    out_i[seg * k + r] = idb[r];
  }
}

// ---------------------------------------------------------------------------
// Rows with k <= 32, pass 1: one warp per kChunkW-column chunk of a row keeps the
// chunk's k best (key, id) sorted across lanes 0..k-1; a batch of 32 elements costs
// one comparison per lane against the running k-th plus a ballot, and the rare
// candidates are inserted with two shuffles.  Pass 2 (topk_segments_kernel) merges
// the per-chunk lists.  Exact: a row's k best are among its chunks' k best.
// ---------------------------------------------------------------------------
constexpr int kChunkW = 8192;
constexpr int kWarpsTk = 8;

__global__ void __launch_bounds__(kWarpsTk * 32)
    topk_rows_chunks_kernel(const float* __restrict__ d, int64_t ld, int64_t n_rows, int64_t row_len,
                            int64_t id_base, int k, int64_t n_chunks, bool vec4, float* __restrict__ cand_d,
                            int64_t* __restrict__ cand_i) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (int64_t)blockIdx.x * kWarpsTk + (threadIdx.x >> 5);
  if (w >= n_rows * n_chunks) return;
  const int64_t row = w / n_chunks, chunk = w - row * n_chunks;
  const int64_t c0 = chunk * kChunkW, c1 = min(row_len, c0 + kChunkW);
  const float* dr = d + row * ld;
  uint32_t my_k = 0xFFFFFFFFu;
  int64_t my_i = INT64_MAX;
  uint32_t thr_k = 0xFFFFFFFFu;
  int64_t thr_i = INT64_MAX;
  auto offer = [&](uint32_t key, int64_t id, bool ok) {
    uint32_t bal = __ballot_sync(0xffffffffu, ok && less(key, id, thr_k, thr_i));
    while (bal) {
      const int src = __ffs(bal) - 1;
      bal &= bal - 1u;
      const uint32_t nk = __shfl_sync(0xffffffffu, key, src);
      const int64_t ni = __shfl_sync(0xffffffffu, id, src);
      if (!less(nk, ni, thr_k, thr_i)) continue;  // the threshold moved since the ballot
      const int pos = __popc(__ballot_sync(0xffffffffu, lane < k && less(my_k, my_i, nk, ni)));
      const uint32_t uk = __shfl_up_sync(0xffffffffu, my_k, 1);
      const int64_t ui = __shfl_up_sync(0xffffffffu, my_i, 1);
      if (lane > pos && lane < k) {
        my_k = uk;
        my_i = ui;
      }
      if (lane == pos) {
        my_k = nk;
        my_i = ni;
      }
      thr_k = __shfl_sync(0xffffffffu, my_k, k - 1);
      thr_i = __shfl_sync(0xffffffffu, my_i, k - 1);
    }
  };
  if (vec4) {  // 16-byte aligned rows: 128 columns per warp step, next step's load in flight
    int64_t c = c0 + lane * 4;
    float4 cur = c + 3 < c1 ? __ldg(reinterpret_cast<const float4*>(dr + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t base = c0; base < c1; base += 128) {
      const int64_t cn = base + 128 + lane * 4;
      const float4 nxt = cn + 3 < c1 ? __ldg(reinterpret_cast<const float4*>(dr + cn)) : make_float4(0.f, 0.f, 0.f, 0.f);
      c = base + lane * 4;
      if (c + 3 >= c1 && c < c1) {  // ragged end of the chunk
        cur.x = dr[c];
        if (c + 1 < c1) cur.y = dr[c + 1];
        if (c + 2 < c1) cur.z = dr[c + 2];
      }
      offer(float_key(cur.x), id_base + c, c < c1);
      offer(float_key(cur.y), id_base + c + 1, c + 1 < c1);
      offer(float_key(cur.z), id_base + c + 2, c + 2 < c1);
      offer(float_key(cur.w), id_base + c + 3, c + 3 < c1);
      cur = nxt;
    }
  } else {
    for (int64_t base = c0; base < c1; base += 32) {
      const int64_t c = base + lane;
      offer(c < c1 ? float_key(dr[c]) : 0xFFFFFFFFu, id_base + c, c < c1);
    }
  }
  if (lane < k) {
    cand_d[w * k + lane] = key_float(my_k);
    cand_i[w * k + lane] = my_i;
  }
}

__global__ void keys_kernel(const float* __restrict__ d, const int64_t* __restrict__ perm, int64_t n,
                            uint32_t* __restrict__ keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    keys[i] = float_key(d[perm ? perm[i] : i]);
}

__global__ void iota_kernel(int64_t* __restrict__ v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) v[i] = i;
}

__global__ void emit_kernel(const float* __restrict__ d, const int64_t* __restrict__ ids,
                            const int64_t* __restrict__ pos_by_id, const int64_t* __restrict__ order, int64_t k,
                            float* __restrict__ out_d, int64_t* __restrict__ out_i) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < k; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = pos_by_id[order[r]];
    out_d[r] = d[p];
    out_i[r] = ids[p];
  }
}

// ---------------------------------------------------------------------------
// Any element type (topk_select keeps the caller's dtype, kernels.py:210-223): an
// order-preserving 64-bit key per element (floats widened exactly to double, -0 == +0,
// NaN last; signed integers with the sign bit flipped; unsigned as is), the same two
// stable radix passes (id, then key), and the k first elements copied back in their
// own type.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t double_key(double d) {
  uint64_t u = (uint64_t)__double_as_longlong(d);
  if ((u & 0x7FFFFFFFFFFFFFFFull) > 0x7FF0000000000000ull) return ~0ull;
  if (u == 0x8000000000000000ull) u = 0ull;
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

__device__ __forceinline__ uint64_t any_key(const void* d, int dtype, int64_t i) {
  switch (dtype) {
    case LCRW_F32: return double_key((double)static_cast<const float*>(d)[i]);
    case LCRW_F64: return double_key(static_cast<const double*>(d)[i]);
    case LCRW_F16: return double_key((double)__half2float(static_cast<const __half*>(d)[i]));
    case LCRW_I8: return (uint64_t)(int64_t)static_cast<const int8_t*>(d)[i] ^ 0x8000000000000000ull;
    case LCRW_I16: return (uint64_t)(int64_t)static_cast<const int16_t*>(d)[i] ^ 0x8000000000000000ull;
    case LCRW_I32: return (uint64_t)(int64_t)static_cast<const int32_t*>(d)[i] ^ 0x8000000000000000ull;
    case LCRW_I64: return (uint64_t)static_cast<const int64_t*>(d)[i] ^ 0x8000000000000000ull;
    case LCRW_U8: return static_cast<const uint8_t*>(d)[i];
    case LCRW_U16: return static_cast<const uint16_t*>(d)[i];
    case LCRW_U32: return static_cast<const uint32_t*>(d)[i];
    default: return static_cast<const uint64_t*>(d)[i];  // LCRW_U64
  }
}

__global__ void keys64_kernel(const void* __restrict__ d, int dtype, const int64_t* __restrict__ perm, int64_t n,
                              uint64_t* __restrict__ keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    keys[i] = any_key(d, dtype, perm[i]);
}

__global__ void emit_any_kernel(const uint8_t* __restrict__ d, int elem, const int64_t* __restrict__ ids,
                                const int64_t* __restrict__ pos_by_id, const int64_t* __restrict__ order, int64_t k,
                                uint8_t* __restrict__ out_d, int64_t* __restrict__ out_i) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < k; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = pos_by_id[order[r]];
    for (int b = 0; b < elem; ++b) out_d[r * elem + b] = d[p * elem + b];
    out_i[r] = ids[p];
  }
}

int dtype_bytes(int dtype) {
  switch (dtype) {
    case LCRW_F16: case LCRW_I16: case LCRW_U16: return 2;
    case LCRW_F32: case LCRW_I32: case LCRW_U32: return 4;
    case LCRW_F64: case LCRW_I64: case LCRW_U64: return 8;
    case LCRW_I8: case LCRW_U8: return 1;
    default: return 0;
  }
}

}  // namespace tk
}  // namespace lcrw

using namespace lcrw;
using namespace lcrw::tk;

extern "C" {

int lcrw_topk_segments(const float* d, const int64_t* ids, int64_t n_seg, int64_t seg_len, int k, float* out_d,
                       int64_t* out_i, void* stream) {
  LCRW_REQUIRE(k >= 1, "k must be >= 1");
  LCRW_REQUIRE(n_seg >= 0 && seg_len >= 0, "lcrw_topk_segments: bad shape");
  if (n_seg == 0 || seg_len == 0) return LCRW_OK;
  if (k > 1024) {
    set_error("lcrw_topk_segments: k=%d > 1024 (use lcrw_topk_sort)", k);
    return LCRW_ERR_UNSUPPORTED;
  }
  LCRW_REQUIRE(d && ids && out_d && out_i, "lcrw_topk_segments: null pointer");
  LCRW_REQUIRE(n_seg < (1ll << 31), "lcrw_topk_segments: too many segments");
  int kp = 1;
  while (kp < k) kp <<= 1;
  topk_segments_kernel<<<(unsigned)n_seg, kThreads, 0, as_stream(stream)>>>(d, ids, seg_len, seg_len, 0, k, kp,
                                                                             out_d, out_i);
  LCRW_CHECK_LAUNCH("topk_segments_kernel");
  return LCRW_OK;
}

static int64_t topk_rows_chunks(int64_t row_len) { return (row_len + kChunkW - 1) / kChunkW; }

int lcrw_topk_rows_workspace(int64_t n_rows, int64_t row_len, int k, size_t* bytes) {
  LCRW_REQUIRE(n_rows >= 0 && row_len >= 0 && k >= 1 && bytes, "lcrw_topk_rows_workspace: bad arguments");
  const size_t n = (size_t)n_rows * topk_rows_chunks(row_len) * k;
  *bytes = (k <= 32 && row_len > 2 * kChunkW) ? (n * 4 + 255) / 256 * 256 + n * 8 : 0;
  return LCRW_OK;
}

int lcrw_topk_rows(const float* d, int64_t ld, int64_t n_rows, int64_t row_len, int64_t id_base, int k,
                   float* out_d, int64_t* out_i, void* ws, size_t ws_bytes, void* stream) {
  LCRW_REQUIRE(k >= 1, "k must be >= 1");
  LCRW_REQUIRE(n_rows >= 0 && row_len >= 0 && ld >= row_len, "lcrw_topk_rows: bad shape");
  if (n_rows == 0 || row_len == 0) return LCRW_OK;
  if (k > 1024) {
    set_error("lcrw_topk_rows: k=%d > 1024", k);
    return LCRW_ERR_UNSUPPORTED;
  }
  LCRW_REQUIRE(d && out_d && out_i, "lcrw_topk_rows: null pointer");
  LCRW_REQUIRE(n_rows < (1ll << 31), "lcrw_topk_rows: too many rows");
  cudaStream_t st = as_stream(stream);
  int kp = 1;
  while (kp < k) kp <<= 1;
  size_t need = 0;
  lcrw_topk_rows_workspace(n_rows, row_len, k, &need);
  if (need == 0) {  // short rows or k > 32: one CTA per row
    topk_segments_kernel<<<(unsigned)n_rows, kThreads, 0, st>>>(d, nullptr, ld, row_len, id_base, k, kp, out_d,
                                                                 out_i);
    LCRW_CHECK_LAUNCH("topk_segments_kernel (rows)");
    return LCRW_OK;
  }
  LCRW_REQUIRE(ws && ws_bytes >= need, "lcrw_topk_rows: workspace too small (use lcrw_topk_rows_workspace)");
  const int64_t n_chunks = topk_rows_chunks(row_len);
  const int64_t n_cand = n_chunks * k;
  float* cand_d = static_cast<float*>(ws);
  int64_t* cand_i = reinterpret_cast<int64_t*>(static_cast<char*>(ws) + ((size_t)n_rows * n_cand * 4 + 255) / 256 * 256);
  const bool vec4 = (ld % 4 == 0) && (reinterpret_cast<uintptr_t>(d) & 15) == 0;
  const int64_t warps = n_rows * n_chunks;
  const int64_t blocks = (warps + kWarpsTk - 1) / kWarpsTk;
  LCRW_REQUIRE(blocks < (1ll << 31), "lcrw_topk_rows: too many chunks");
  {
    ProfScope prof(st, "topk_rows");
    topk_rows_chunks_kernel<<<(unsigned)blocks, kWarpsTk * 32, 0, st>>>(d, ld, n_rows, row_len, id_base, k, n_chunks,
                                                                        vec4, cand_d, cand_i);
    LCRW_CHECK_LAUNCH("topk_rows_chunks_kernel");
    topk_segments_kernel<<<(unsigned)n_rows, kThreads, 0, st>>>(cand_d, cand_i, n_cand, n_cand, 0, k, kp, out_d,
                                                                 out_i);
    LCRW_CHECK_LAUNCH("topk_segments_kernel (chunk merge)");
  }
  return LCRW_OK;
}

static size_t align256(size_t x) { return (x + 255) / 256 * 256; }

int lcrw_topk_sort_workspace(int64_t n, size_t* bytes) {
  LCRW_REQUIRE(n >= 0 && bytes, "lcrw_topk_sort_workspace: bad arguments");
  size_t c1 = 0, c2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, c1, (const int64_t*)nullptr, (int64_t*)nullptr, (const int64_t*)nullptr,
                                  (int64_t*)nullptr, (int64_t)n);
  cub::DeviceRadixSort::SortPairs(nullptr, c2, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const int64_t*)nullptr, (int64_t*)nullptr, (int64_t)n);
  // sorted ids, iota/positions, positions by id, keys in/out, rank iota, order
  *bytes = 6 * align256((size_t)n * 8) + (c1 > c2 ? c1 : c2);
  return LCRW_OK;
}

// Two stable radix passes: by id, then by distance key -> lexicographic (distance, id).
int lcrw_topk_sort(const float* d, const int64_t* ids, int64_t n, int64_t k, float* out_d, int64_t* out_i, void* ws,
                   size_t ws_bytes, void* stream) {
  LCRW_REQUIRE(k >= 1, "k must be >= 1");
  LCRW_REQUIRE(n >= 0, "lcrw_topk_sort: bad shape");
  if (n == 0) return LCRW_OK;
  LCRW_REQUIRE(d && ids && out_d && out_i && ws, "lcrw_topk_sort: null pointer");
  size_t need = 0;
  lcrw_topk_sort_workspace(n, &need);
  LCRW_REQUIRE(ws_bytes >= need, "lcrw_topk_sort: workspace too small");
  cudaStream_t st = as_stream(stream);
  char* p = static_cast<char*>(ws);
  const size_t a = align256((size_t)n * 8);
  int64_t* ids_sorted = reinterpret_cast<int64_t*>(p);
  int64_t* pos = reinterpret_cast<int64_t*>(p + a);
  int64_t* pos_sorted = reinterpret_cast<int64_t*>(p + 2 * a);
  uint32_t* keys = reinterpret_cast<uint32_t*>(p + 3 * a);
  uint32_t* keys_sorted = reinterpret_cast<uint32_t*>(p + 4 * a);
  int64_t* rank = reinterpret_cast<int64_t*>(p + 5 * a);
  int64_t* order = ids_sorted;  // reused after pass 1
  void* cub_ws = p + 6 * a;
  size_t cub_bytes = need - 6 * a;
  const unsigned g = (unsigned)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096);
  iota_kernel<<<g, 256, 0, st>>>(pos, n);
  cudaError_t e = cub::DeviceRadixSort::SortPairs(cub_ws, cub_bytes, ids, ids_sorted, pos, pos_sorted, n, 0, 64, st);
  if (e != cudaSuccess) return cuda_status(e, "cub SortPairs (ids)");
  keys_kernel<<<g, 256, 0, st>>>(d, pos_sorted, n, keys);
  iota_kernel<<<g, 256, 0, st>>>(rank, n);
  e = cub::DeviceRadixSort::SortPairs(cub_ws, cub_bytes, keys, keys_sorted, rank, order, n, 0, 32, st);
  if (e != cudaSuccess) return cuda_status(e, "cub SortPairs (keys)");
  const int64_t kk = k < n ? k : n;
  emit_kernel<<<g, 256, 0, st>>>(d, ids, pos_sorted, order, kk, out_d, out_i);
  LCRW_CHECK_LAUNCH("topk emit");
  return LCRW_OK;
}

int lcrw_topk_sort_any_workspace(int64_t n, size_t* bytes) {
  LCRW_REQUIRE(n >= 0 && bytes, "lcrw_topk_sort_any_workspace: bad arguments");
  size_t c1 = 0, c2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, c1, (const int64_t*)nullptr, (int64_t*)nullptr, (const int64_t*)nullptr,
                                  (int64_t*)nullptr, (int64_t)n);
  cub::DeviceRadixSort::SortPairs(nullptr, c2, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                  (const int64_t*)nullptr, (int64_t*)nullptr, (int64_t)n);
  // sorted ids, positions, positions by id, keys in/out, rank iota
  *bytes = 6 * align256((size_t)n * 8) + (c1 > c2 ? c1 : c2);
  return LCRW_OK;
}

// topk_select for distances of any numeric dtype (LCRW_F32 .. LCRW_U64): the k smallest
// under ascending (distance, id), distances copied back in their own type.
int lcrw_topk_sort_any(const void* d, int dtype, const int64_t* ids, int64_t n, int64_t k, void* out_d,
                       int64_t* out_i, void* ws, size_t ws_bytes, void* stream) {
  LCRW_REQUIRE(k >= 1, "k must be >= 1");
  LCRW_REQUIRE(n >= 0, "lcrw_topk_sort_any: bad shape");
  const int elem = dtype_bytes(dtype);
  LCRW_REQUIRE(elem > 0, "lcrw_topk_sort_any: unsupported dtype code");
  if (n == 0) return LCRW_OK;
  LCRW_REQUIRE(d && ids && out_d && out_i && ws, "lcrw_topk_sort_any: null pointer");
  size_t need = 0;
  lcrw_topk_sort_any_workspace(n, &need);
  LCRW_REQUIRE(ws_bytes >= need, "lcrw_topk_sort_any: workspace too small");
  cudaStream_t st = as_stream(stream);
  char* p = static_cast<char*>(ws);
  const size_t a = align256((size_t)n * 8);
  int64_t* ids_sorted = reinterpret_cast<int64_t*>(p);
  int64_t* pos = reinterpret_cast<int64_t*>(p + a);
  int64_t* pos_sorted = reinterpret_cast<int64_t*>(p + 2 * a);
  uint64_t* keys = reinterpret_cast<uint64_t*>(p + 3 * a);
  uint64_t* keys_sorted = reinterpret_cast<uint64_t*>(p + 4 * a);
  int64_t* rank = reinterpret_cast<int64_t*>(p + 5 * a);
  int64_t* order = ids_sorted;  // reused after pass 1
  void* cub_ws = p + 6 * a;
  size_t cub_bytes = need - 6 * a;
  const unsigned g = (unsigned)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096);
  iota_kernel<<<g, 256, 0, st>>>(pos, n);
  cudaError_t e = cub::DeviceRadixSort::SortPairs(cub_ws, cub_bytes, ids, ids_sorted, pos, pos_sorted, n, 0, 64, st);
  if (e != cudaSuccess) return cuda_status(e, "cub SortPairs (ids)");
  keys64_kernel<<<g, 256, 0, st>>>(d, dtype, pos_sorted, n, keys);
  iota_kernel<<<g, 256, 0, st>>>(rank, n);
  e = cub::DeviceRadixSort::SortPairs(cub_ws, cub_bytes, keys, keys_sorted, rank, order, n, 0, 64, st);
  if (e != cudaSuccess) return cuda_status(e, "cub SortPairs (keys)");
  const int64_t kk = k < n ? k : n;
  emit_any_kernel<<<g, 256, 0, st>>>(static_cast<const uint8_t*>(d), elem, ids, pos_sorted, order, kk,
                                     static_cast<uint8_t*>(out_d), out_i);
  LCRW_CHECK_LAUNCH("topk emit (any dtype)");
  return LCRW_OK;
}

}  // extern "C"
