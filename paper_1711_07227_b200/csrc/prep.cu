// Operand preparation, vocabulary restriction, exact-identity classes and the
// segment plan for Phase 1.  All memory-bound one-pass kernels; CUB supplies
// the scan / radix sort plumbing.
#include <cub/cub.cuh>

#include "common.cuh"

namespace lcrw {
namespace {

constexpr int kThreads = 256;

inline unsigned grid_for(int64_t n, int threads = kThreads, int64_t cap = 148 * 32) {
  int64_t g = ceil_div(n, threads);
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<unsigned>(g);
}

// ---------------------------------------------------------------------------
// scale selection and f16 operand rows
// ---------------------------------------------------------------------------
// max over rows of |x_r|^2 (fp32), atomically max-accumulated as float bits
__global__ void max_sqnorm_kernel(const float* __restrict__ x, int64_t rows, int m, uint32_t* out) {
  const int lane = threadIdx.x & 31;
  float best = 0.f;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < rows;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    float acc = 0.f;
    for (int k = lane; k < m; k += 32) {
      const float v = x[r * (int64_t)m + k];
      acc = fmaf(v, v, acc);
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    best = fmaxf(best, acc);
  }
  if (lane == 0 && best > 0.f) atomicMax(out, __float_as_uint(best));
}

// s = 2^k with s^2 * max|x|^2 in [2^12, 2^14): scaled squared norms (and their
// three-piece f16 split) fit f16, scaled elements are <= 2^7
__global__ void scale_kernel(const uint32_t* max_bits, float* scale) {
  const float a = __uint_as_float(*max_bits);
  int k = 0;
  if (a > 0.f && isfinite(a)) {
    int e;
    frexpf(a, &e);  // a in [2^(e-1), 2^e)
    k = (14 - e) >> 1;  // floor((14 - e) / 2): 2k + e <= 14
    k = max(-60, min(60, k));
  }
  scale[0] = ldexpf(1.f, k);
  scale[1] = ldexpf(1.f, -k);
}

// one warp per row.  With x' = scale * x, hi = f16(x'), lo = f16(x' - hi):
//   layout 0 (A)        [hi(x')                         , 1, 1, 1]          K = m + 3
//   layout 1 (A split)  [hi, hi, lo                     , 1, 1, 1]          K = 3m + 3
//   layout 2 (B)        [-2 hi(x')                      , n_hi, n_mid, n_lo] K = m + 3
//   layout 3 (B split)  [-2 hi, -2 lo, -2 hi            , n_hi, n_mid, n_lo] K = 3m + 3
// n = |rounded row|^2 (fp64 sum) split into three f16 pieces, so one MMA dot of
// an A row with a B row is |b|^2 - 2 a.b and the Gram expansion needs only
// +|a|^2 per segment in the epilogue.  norms[r] = n (f32), used for the A side.
__global__ void prepare_rows_kernel(const float* __restrict__ X, int64_t rows, int m, int kp, int layout,
                                    const float* __restrict__ scale, __half* __restrict__ Xh,
                                    float* __restrict__ norms) {
  const int lane = threadIdx.x & 31;
  const float s = scale[0];
  const bool split = layout & 1;
  const bool bside = layout & 2;
  const int k_vec = split ? 3 * m : m;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < rows;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const float* src = X + r * (int64_t)m;
    __half* dst = Xh + r * (int64_t)kp;
    double acc = 0.0;
    for (int c = lane; c < m; c += 32) {
      const float x = src[c] * s;
      const __half hi = __float2half_rn(x);
      const double v = split ? (double)__half2float(hi) + (double)__half2float(__float2half_rn(x - __half2float(hi)))
                             : (double)__half2float(hi);
      acc += v * v;
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    const float n_hi = __half2float(__float2half_rn((float)acc));
    const double r1 = acc - (double)n_hi;
    const float n_mid = __half2float(__float2half_rn((float)r1));
    const float n_lo = (float)(r1 - (double)n_mid);
    for (int k = lane; k < kp; k += 32) {
      float out = 0.f;
      if (k < k_vec) {
        const int part = split ? k / m : 0;
        const int c = k - part * m;
        const float x = src[c] * s;
        const __half hi = __float2half_rn(x);
        const bool want_lo = split && ((!bside && part == 2) || (bside && part == 1));
        const float val = want_lo ? __half2float(__float2half_rn(x - __half2float(hi))) : __half2float(hi);
        out = bside ? -2.f * val : val;
      } else if (k < k_vec + 3) {
        const int t = k - k_vec;
        out = bside ? (t == 0 ? n_hi : t == 1 ? n_mid : n_lo) : 1.f;
      }
      dst[k] = __float2half_rn(out);
    }
    if (lane == 0 && norms) norms[r] = (float)acc;
  }
}

// one warp per output row: 16-byte vector copies of kp f16 values.
__global__ void gather_rows_kernel(const int4* __restrict__ Xh, const float* __restrict__ norms, int vec_per_row,
                                   const int32_t* __restrict__ ids, int64_t n, int4* __restrict__ T,
                                   float* __restrict__ tnorms) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < n;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t g = ids[i];
    const int4* src = Xh + g * vec_per_row;
    int4* dst = T + i * vec_per_row;
    for (int v = lane; v < vec_per_row; v += 32) dst[v] = __ldg(src + v);
    if (lane == 0 && tnorms) tnorms[i] = norms[g];
  }
}

// ---------------------------------------------------------------------------
// exact-identity classes (bitwise-equal fp32 rows, +0 == -0)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t canon_bits(float x) { return x == 0.f ? 0u : __float_as_uint(x); }

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// order-independent per-element mix, summed across the warp
__global__ void hash_rows_kernel(const float* __restrict__ X, int64_t rows, int m, uint64_t* __restrict__ h,
                                 int32_t* __restrict__ ids) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < rows;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    uint64_t acc = 0;
    for (int k = lane; k < m; k += 32)
      acc += mix64((static_cast<uint64_t>(k) << 32) ^ canon_bits(X[r * (int64_t)m + k]) ^ 0x9e3779b97f4a7c15ull);
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      h[r] = mix64(acc);
      if (ids) ids[r] = static_cast<int32_t>(r);
    }
  }
}

__device__ bool rows_equal(const float* __restrict__ a, const float* __restrict__ b, int m) {
  for (int k = 0; k < m; ++k)
    if (canon_bits(a[k]) != canon_bits(b[k])) return false;
  return true;
}

// position i of the (hash, id)-sorted order: smallest identical id in the run
__global__ void canon_kernel(const float* __restrict__ E, int64_t rows, int m, const uint64_t* __restrict__ sh,
                             const int32_t* __restrict__ sid, int32_t* __restrict__ canon,
                             unsigned long long* n_dup) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t id = sid[i];
    int32_t c = id;
    int64_t j = i;
    while (j > 0 && sh[j - 1] == sh[i]) --j;  // run start
    for (; j < i; ++j) {
      if (rows_equal(E + (int64_t)sid[j] * m, E + (int64_t)id * m, m)) {
        c = sid[j];
        break;
      }
    }
    canon[id] = c;
    if (c != id) atomicAdd(n_dup, 1ull);
  }
}

__global__ void next_kernel(int64_t rows, const uint64_t* __restrict__ sh, const int32_t* __restrict__ sid,
                            const int32_t* __restrict__ canon, int32_t* __restrict__ next) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t id = sid[i];
    int32_t nx = -1;
    for (int64_t j = i + 1; j < rows && sh[j] == sh[i]; ++j) {
      if (canon[sid[j]] == canon[id]) {
        nx = sid[j];
        break;
      }
    }
    next[id] = nx;
  }
}

__global__ void match_kernel(const float* __restrict__ Q, int64_t nq, const float* __restrict__ E, int m,
                             const uint64_t* __restrict__ qh, const uint64_t* __restrict__ sh,
                             const int32_t* __restrict__ sid, int64_t rows, const int32_t* __restrict__ canon,
                             int32_t* __restrict__ rep) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nq; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t h = qh[i];
    int64_t lo = 0, hi = rows;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (sh[mid] < h) lo = mid + 1; else hi = mid;
    }
    int32_t r = -1;
    for (int64_t j = lo; j < rows && sh[j] == h; ++j) {
      if (rows_equal(E + (int64_t)sid[j] * m, Q + i * (int64_t)m, m)) {
        r = canon[sid[j]];
        break;
      }
    }
    rep[i] = r;
  }
}

// ---------------------------------------------------------------------------
// restriction (corpus.py:405-426)
// ---------------------------------------------------------------------------
__global__ void mark_kernel(const int32_t* __restrict__ cols, int64_t nnz, int32_t* __restrict__ flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x)
    flags[cols[i]] = 1;
}

__global__ void finalize_remap_kernel(const int32_t* __restrict__ flags, int64_t n, int32_t* __restrict__ remap,
                                      int32_t* __restrict__ used, int64_t* n_used) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
    const int32_t pos = remap[c];  // exclusive scan
    if (c == n - 1) *n_used = (int64_t)pos + flags[c];
    if (flags[c]) {
      used[pos] = static_cast<int32_t>(c);
    } else {
      remap[c] = -1;
    }
  }
}

__global__ void remap_ids_kernel(const int32_t* __restrict__ cols, int64_t nnz, const int32_t* __restrict__ remap,
                                 int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = remap[cols[i]];
}

// ---------------------------------------------------------------------------
// Phase-1 segment plan and exact zeros
// ---------------------------------------------------------------------------
__global__ void endmask_kernel(const int64_t* __restrict__ offs, int64_t base, int64_t n_seg,
                               uint32_t* __restrict__ mask) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n_seg; s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t last = offs[s + 1] - 1 - base;
    atomicOr(mask + (last >> 5), 1u << (last & 31));
  }
}

__global__ void ranges_kernel(const int64_t* __restrict__ offs, int64_t base, int64_t n_seg, int range_cols,
                              int32_t* __restrict__ range_seg, int64_t n_ranges) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= n_ranges; r += (int64_t)gridDim.x * blockDim.x) {
    if (r == n_ranges) {
      range_seg[r] = static_cast<int32_t>(n_seg);
      continue;
    }
    const int64_t target = r * (int64_t)range_cols;
    int64_t lo = 0, hi = n_seg;  // first s in [0, n_seg] with offs[s] >= target
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (offs[mid] - base < target) lo = mid + 1; else hi = mid;
    }
    range_seg[r] = static_cast<int32_t>(lo);
  }
}

// one warp per segment, lanes over its B rows (rep indexed by the raw offsets)
__global__ void zero_identical_kernel(const int64_t* __restrict__ offs, int64_t n_seg, const int32_t* __restrict__ rep,
                                      const int32_t* __restrict__ next, const int32_t* __restrict__ remap,
                                      float* __restrict__ Z, int64_t z_panel, int z_shift) {
  const int lane = threadIdx.x & 31;
  const int64_t zmask = (1ll << z_shift) - 1;
  for (int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; s < n_seg;
       s += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    float* zs = Z + (s >> z_shift) * z_panel + (s & zmask);
    for (int64_t t = offs[s] + lane; t < offs[s + 1]; t += 32) {
      for (int32_t g = rep[t]; g >= 0; g = next ? next[g] : -1) {
        const int32_t r = remap ? remap[g] : g;
        if (r >= 0) zs[(int64_t)r << z_shift] = 0.f;
      }
    }
  }
}

}  // namespace
}  // namespace lcrw

using namespace lcrw;

extern "C" {

int lcrw_max_sqnorm(const float* x, int64_t rows, int m, uint32_t* max_bits, void* stream) {
  LCRW_REQUIRE(rows >= 0 && m > 0 && (rows == 0 || x) && max_bits, "lcrw_max_sqnorm: bad arguments");
  if (rows == 0) return LCRW_OK;
  max_sqnorm_kernel<<<grid_for(rows * 32), kThreads, 0, as_stream(stream)>>>(x, rows, m, max_bits);
  LCRW_CHECK_LAUNCH("max_sqnorm_kernel");
  return LCRW_OK;
}

int lcrw_scale_from_max_sqnorm(const uint32_t* max_bits, float* scale, void* stream) {
  LCRW_REQUIRE(max_bits && scale, "lcrw_scale_from_max_sqnorm: null pointer");
  scale_kernel<<<1, 1, 0, as_stream(stream)>>>(max_bits, scale);
  LCRW_CHECK_LAUNCH("scale_kernel");
  return LCRW_OK;
}

int lcrw_prepare_rows(const float* X, int64_t rows, int m, int kp, int layout, const float* scale, uint16_t* Xh,
                      float* norms, void* stream) {
  LCRW_REQUIRE(layout >= 0 && layout <= 3, "lcrw_prepare_rows: layout must be 0..3");
  LCRW_REQUIRE(rows >= 0 && m > 0 && kp == lcrw_padded_dim(lcrw_operand_k(m, layout & 1)),
               "lcrw_prepare_rows: bad shape");
  LCRW_REQUIRE(rows == 0 || (X && scale && Xh), "lcrw_prepare_rows: null pointer");
  if (rows == 0) return LCRW_OK;
  prepare_rows_kernel<<<grid_for(rows * 32), kThreads, 0, as_stream(stream)>>>(
      X, rows, m, kp, layout, scale, reinterpret_cast<__half*>(Xh), norms);
  LCRW_CHECK_LAUNCH("prepare_rows_kernel");
  return LCRW_OK;
}

int lcrw_gather_rows(const uint16_t* Xh, const float* norms, int kp, const int32_t* ids, int64_t n, uint16_t* T,
                     float* tnorms, void* stream) {
  LCRW_REQUIRE(n >= 0 && kp > 0 && kp % 64 == 0, "lcrw_gather_rows: bad shape");
  if (n == 0) return LCRW_OK;
  LCRW_REQUIRE(Xh && ids && T && (norms || !tnorms), "lcrw_gather_rows: null pointer");
  gather_rows_kernel<<<grid_for(n * 32), kThreads, 0, as_stream(stream)>>>(
      reinterpret_cast<const int4*>(Xh), norms, kp / 8, ids, n, reinterpret_cast<int4*>(T), tnorms);
  LCRW_CHECK_LAUNCH("gather_rows_kernel");
  return LCRW_OK;
}

int lcrw_row_classes_workspace(int64_t rows, size_t* bytes) {
  LCRW_REQUIRE(rows >= 0 && bytes, "lcrw_row_classes_workspace: bad arguments");
  size_t cub_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, (int64_t)rows);
  // hashes + ids (unsorted) + n_dup counter + cub scratch
  *bytes = ((size_t)rows * 12 + 255) / 256 * 256 + 256 + cub_bytes;
  return LCRW_OK;
}

int lcrw_row_classes(const float* E, int64_t rows, int m, int32_t* canon, int32_t* next, int64_t* n_dup,
                     uint64_t* sorted_hash, int32_t* sorted_ids, void* ws, size_t ws_bytes, void* stream) {
  LCRW_REQUIRE(rows >= 0 && m > 0, "lcrw_row_classes: bad shape");
  LCRW_REQUIRE(rows == 0 || (E && canon && next && n_dup && sorted_hash && sorted_ids && ws),
               "lcrw_row_classes: null pointer");
  size_t need = 0;
  lcrw_row_classes_workspace(rows, &need);
  LCRW_REQUIRE(ws_bytes >= need, "lcrw_row_classes: workspace too small");
  cudaStream_t st = as_stream(stream);
  if (rows == 0) return LCRW_OK;
  char* p = static_cast<char*>(ws);
  uint64_t* h = reinterpret_cast<uint64_t*>(p);
  int32_t* ids = reinterpret_cast<int32_t*>(p + rows * 8);
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(p + ((size_t)rows * 12 + 255) / 256 * 256);
  void* cub_ws = p + ((size_t)rows * 12 + 255) / 256 * 256 + 256;
  size_t cub_bytes = need - (((size_t)rows * 12 + 255) / 256 * 256 + 256);
  cudaMemsetAsync(cnt, 0, 8, st);
  hash_rows_kernel<<<grid_for(rows * 32), kThreads, 0, st>>>(E, rows, m, h, ids);
  LCRW_CHECK_LAUNCH("hash_rows_kernel");
  cudaError_t e = cub::DeviceRadixSort::SortPairs(cub_ws, cub_bytes, h, sorted_hash, ids, sorted_ids, rows, 0, 64, st);
  if (e != cudaSuccess) return cuda_status(e, "cub SortPairs (row classes)");
  canon_kernel<<<grid_for(rows), kThreads, 0, st>>>(E, rows, m, sorted_hash, sorted_ids, canon, cnt);
  LCRW_CHECK_LAUNCH("canon_kernel");
  next_kernel<<<grid_for(rows), kThreads, 0, st>>>(rows, sorted_hash, sorted_ids, canon, next);
  LCRW_CHECK_LAUNCH("next_kernel");
  e = cudaMemcpyAsync(n_dup, cnt, 8, cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return cuda_status(e, "copy n_dup");
  return LCRW_OK;
}

int lcrw_match_rows(const float* Q, int64_t nq, const float* E, int m, const uint64_t* sorted_hash,
                    const int32_t* sorted_ids, int64_t rows, const int32_t* canon, int32_t* rep, void* stream) {
  LCRW_REQUIRE(nq >= 0 && m > 0 && rows >= 0, "lcrw_match_rows: bad shape");
  if (nq == 0) return LCRW_OK;
  LCRW_REQUIRE(Q && E && sorted_hash && sorted_ids && canon && rep, "lcrw_match_rows: null pointer");
  cudaStream_t st = as_stream(stream);
  uint64_t* qh = nullptr;
  cudaError_t e = cudaMallocAsync(&qh, nq * 8, st);
  if (e != cudaSuccess) return cuda_status(e, "cudaMallocAsync (match hashes)");
  hash_rows_kernel<<<grid_for(nq * 32), kThreads, 0, st>>>(Q, nq, m, qh, nullptr);
  match_kernel<<<grid_for(nq), kThreads, 0, st>>>(Q, nq, E, m, qh, sorted_hash, sorted_ids, rows, canon, rep);
  cudaError_t le = cudaGetLastError();
  cudaFreeAsync(qh, st);
  if (le != cudaSuccess) return cuda_status(le, "match_kernel");
  return LCRW_OK;
}

int lcrw_restrict_workspace(int64_t n_cols, size_t* bytes) {
  LCRW_REQUIRE(n_cols >= 0 && bytes, "lcrw_restrict_workspace: bad arguments");
  size_t cub_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, cub_bytes, (const int32_t*)nullptr, (int32_t*)nullptr, (int64_t)n_cols);
  *bytes = ((size_t)n_cols * 4 + 255) / 256 * 256 + cub_bytes;
  return LCRW_OK;
}

int lcrw_restrict(const int32_t* col_ids, int64_t nnz, int64_t n_cols, int32_t* remap, int32_t* used,
                  int64_t* n_used, void* ws, size_t ws_bytes, void* stream) {
  LCRW_REQUIRE(nnz >= 0 && n_cols > 0, "lcrw_restrict: bad shape");
  LCRW_REQUIRE(remap && used && n_used && ws && (nnz == 0 || col_ids), "lcrw_restrict: null pointer");
  size_t need = 0;
  lcrw_restrict_workspace(n_cols, &need);
  LCRW_REQUIRE(ws_bytes >= need, "lcrw_restrict: workspace too small");
  cudaStream_t st = as_stream(stream);
  int32_t* flags = static_cast<int32_t*>(ws);
  const size_t off = ((size_t)n_cols * 4 + 255) / 256 * 256;
  size_t cub_bytes = need - off;
  cudaMemsetAsync(flags, 0, n_cols * 4, st);
  if (nnz) {
    mark_kernel<<<grid_for(nnz), kThreads, 0, st>>>(col_ids, nnz, flags);
    LCRW_CHECK_LAUNCH("mark_kernel");
  }
  cudaError_t e = cub::DeviceScan::ExclusiveSum(static_cast<char*>(ws) + off, cub_bytes, flags, remap, n_cols, st);
  if (e != cudaSuccess) return cuda_status(e, "cub ExclusiveSum (restrict)");
  finalize_remap_kernel<<<grid_for(n_cols), kThreads, 0, st>>>(flags, n_cols, remap, used, n_used);
  LCRW_CHECK_LAUNCH("finalize_remap_kernel");
  return LCRW_OK;
}

int lcrw_remap_ids(const int32_t* col_ids, int64_t nnz, const int32_t* remap, int32_t* out, void* stream) {
  LCRW_REQUIRE(nnz >= 0, "lcrw_remap_ids: bad shape");
  if (nnz == 0) return LCRW_OK;
  LCRW_REQUIRE(col_ids && remap && out, "lcrw_remap_ids: null pointer");
  remap_ids_kernel<<<grid_for(nnz), kThreads, 0, as_stream(stream)>>>(col_ids, nnz, remap, out);
  LCRW_CHECK_LAUNCH("remap_ids_kernel");
  return LCRW_OK;
}

int64_t lcrw_endmask_words(int64_t n_cols) { return (n_cols + 320) / 32; }

int64_t lcrw_plan_ranges(int64_t n_cols, int range_cols) {
  if (range_cols <= 0) return -1;
  int64_t n = ceil_div(n_cols, range_cols);
  return n < 1 ? 1 : n;
}

int lcrw_segment_plan(const int64_t* seg_offsets, int64_t seg_base, int64_t n_seg, int64_t n_cols, int range_cols,
                      uint32_t* endmask, int32_t* range_seg, int64_t n_ranges, void* stream) {
  LCRW_REQUIRE(n_seg >= 1 && n_cols >= n_seg && range_cols > 0 && n_ranges >= 1, "lcrw_segment_plan: bad shape");
  LCRW_REQUIRE(seg_offsets && endmask && range_seg, "lcrw_segment_plan: null pointer");
  cudaStream_t st = as_stream(stream);
  cudaMemsetAsync(endmask, 0, lcrw_endmask_words(n_cols) * 4, st);
  endmask_kernel<<<grid_for(n_seg), kThreads, 0, st>>>(seg_offsets, seg_base, n_seg, endmask);
  LCRW_CHECK_LAUNCH("endmask_kernel");
  ranges_kernel<<<grid_for(n_ranges + 1), kThreads, 0, st>>>(seg_offsets, seg_base, n_seg, range_cols, range_seg,
                                                             n_ranges);
  LCRW_CHECK_LAUNCH("ranges_kernel");
  return LCRW_OK;
}

int lcrw_zero_identical(const int64_t* seg_offsets, int64_t n_seg, const int32_t* rep, const int32_t* next,
                        const int32_t* remap, float* Z, int64_t z_panel, int z_shift, void* stream) {
  LCRW_REQUIRE(n_seg >= 0, "lcrw_zero_identical: bad shape");
  if (n_seg == 0) return LCRW_OK;
  LCRW_REQUIRE(seg_offsets && rep && Z, "lcrw_zero_identical: null pointer");
  LCRW_REQUIRE(z_shift >= 0 && z_shift <= 10, "lcrw_zero_identical: z_shift out of range");
  zero_identical_kernel<<<grid_for(n_seg * 32), kThreads, 0, as_stream(stream)>>>(seg_offsets, n_seg, rep, next,
                                                                                 remap, Z, z_panel, z_shift);
  LCRW_CHECK_LAUNCH("zero_identical_kernel");
  return LCRW_OK;
}

}  // extern "C"
