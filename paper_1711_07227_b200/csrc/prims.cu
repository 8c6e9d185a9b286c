// Reference compute primitives that sit next to the hot path and are part of the
// drop-in surface of movers.kernels (kernels.py:66-167): squared_norms,
// euclidean_into, row_min / col_min, segmented_min.
//
// squared_norms / euclidean_into reproduce the reference BIT FOR BIT: float64
// products, numpy's pairwise summation over the contiguous m axis
// (np.sum(..., axis=-1): blocks of 8 partial sums up to 128 elements, halving
// above), then sq = (|a|^2 + |b|^2) - 2 dot, clamp at 0, IEEE sqrt, one rounding
// to f32 (kernels.py:105-109).  Every operation is an explicit _rn intrinsic, so
// nothing is contracted into an FMA.  These are the fp64 primitives, not the
// f16 tensor-core Phase 1 of the hot path (phase1.cu), whose error budget is
// stated in DESIGN.md.
//
// The minima follow numpy's np.minimum semantics in the reduction order numpy
// uses (left to right): acc = (acc < x || acc != acc) ? acc : x -- NaN propagates.
#include "common.cuh"

namespace lcrw {
namespace prims {

constexpr int kPwBlock = 128;  // numpy PW_BLOCKSIZE

inline unsigned grid_for(int64_t n, int threads = 256, int64_t cap = 148 * 32) {
  const int64_t b = (n + threads - 1) / threads;
  return (unsigned)(b < 1 ? 1 : (b > cap ? cap : b));
}

// numpy's pairwise_sum of f(i), i in [0, n), for n <= kPwBlock
template <class F>
__device__ __forceinline__ double pw_block(F f, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r = __dadd_rn(r, f(i));
    return r;
  }
  double r0 = f(0), r1 = f(1), r2 = f(2), r3 = f(3), r4 = f(4), r5 = f(5), r6 = f(6), r7 = f(7);
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8) {
    r0 = __dadd_rn(r0, f(i + 0));
    r1 = __dadd_rn(r1, f(i + 1));
    r2 = __dadd_rn(r2, f(i + 2));
    r3 = __dadd_rn(r3, f(i + 3));
    r4 = __dadd_rn(r4, f(i + 4));
    r5 = __dadd_rn(r5, f(i + 5));
    r6 = __dadd_rn(r6, f(i + 6));
    r7 = __dadd_rn(r7, f(i + 7));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r0, r1), __dadd_rn(r2, r3)),
                         __dadd_rn(__dadd_rn(r4, r5), __dadd_rn(r6, r7)));
  for (; i < n; ++i) res = __dadd_rn(res, f(i));
  return res;
}

// numpy's pairwise_sum for any n: the recursion (split n2 = n/2 - (n/2) % 8) walked with an
// explicit stack; partial sums combine in the recursion's order
template <class F>
__device__ double pairwise_sum(F f, int64_t n) {
  if (n <= kPwBlock) return pw_block(f, n);
  // frames: (start, len, state) -- state 0: not expanded, 1: left done (value in vals)
  int64_t st_start[40], st_len[40];
  double st_left[40];
  int st_state[40];
  int top = 0;
  st_start[0] = 0;
  st_len[0] = n;
  st_state[0] = 0;
  double ret = 0.0;
  bool have_ret = false;
  while (top >= 0) {
    const int64_t s = st_start[top], len = st_len[top];
    if (have_ret) {  // a child returned into frame `top`
      have_ret = false;
      if (st_state[top] == 1) {  // left child done: descend right
        st_left[top] = ret;
        st_state[top] = 2;
        int64_t n2 = len / 2;
        n2 -= n2 % 8;
        ++top;
        st_start[top] = s + n2;
        st_len[top] = len - n2;
        st_state[top] = 0;
        continue;
      }
      ret = __dadd_rn(st_left[top], ret);  // right child done
      have_ret = true;
      --top;
      continue;
    }
    if (len <= kPwBlock) {
      ret = pw_block([&](int64_t i) { return f(s + i); }, len);
      have_ret = true;
      --top;
      continue;
    }
    int64_t n2 = len / 2;
    n2 -= n2 % 8;
    st_state[top] = 1;
    ++top;
    st_start[top] = s;
    st_len[top] = n2;
    st_state[top] = 0;
  }
  return ret;
}

template <class T>
__device__ __forceinline__ double as_f64(T v) {
  return (double)v;
}

__global__ void squared_norms_kernel(const float* __restrict__ a, int64_t rows, int64_t m, double* __restrict__ out) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    const float* row = a + r * m;
    out[r] = pairwise_sum(
        [&](int64_t i) {
          const double x = (double)row[i];
          return __dmul_rn(x, x);
        },
        m);
  }
}

__global__ void squared_norms64_kernel(const double* __restrict__ a, int64_t rows, int64_t m,
                                       double* __restrict__ out) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    const double* row = a + r * m;
    out[r] = pairwise_sum([&](int64_t i) { return __dmul_rn(row[i], row[i]); }, m);
  }
}

// out[i, j] (row stride ld) = f32(sqrt(max(0, (sq_a[i] + sq_b[j]) - 2 * dot(a_i, b_j)))), kernels.py:105-109
__global__ void __launch_bounds__(256) euclidean_kernel(const double* __restrict__ a, const double* __restrict__ sq_a,
                                                        int64_t r, const double* __restrict__ b,
                                                        const double* __restrict__ sq_b, int64_t c, int64_t m,
                                                        void* __restrict__ out, int64_t ld, int out_f64) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t i = blockIdx.y;
  if (j >= c || i >= r) return;
  const double* ar = a + i * m;
  const double* br = b + j * m;
  const double dot = pairwise_sum([&](int64_t t) { return __dmul_rn(ar[t], br[t]); }, m);
  double sq = __dsub_rn(__dadd_rn(sq_a[i], sq_b[j]), __dmul_rn(2.0, dot));
  sq = (sq > 0.0 || sq != sq) ? sq : 0.0;  // np.maximum(sq, 0.0): NaN stays NaN
  const double d = __dsqrt_rn(sq);
  if (out_f64)
    static_cast<double*>(out)[i * ld + j] = d;  // an f64 `out` keeps the f64 values (kernels.py:109)
  else
    static_cast<float*>(out)[i * ld + j] = (float)d;
}

template <class T>
__device__ __forceinline__ T np_min(T acc, T x) {
  return (acc < x || acc != acc) ? acc : x;
}

// reduce over the middle axis of an (outer, n, inner) array, segments [seg[s], seg[s+1]) of it:
// out[o, s, k] = minimum.reduce(v[o, seg[s]:seg[s+1], k]) (left to right)
template <class T>
__global__ void segmin_kernel(const T* __restrict__ v, int64_t outer, int64_t n, int64_t inner,
                              const int64_t* __restrict__ seg, int64_t n_seg, T* __restrict__ out) {
  const int64_t total = outer * n_seg * inner;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = t % inner, rest = t / inner, s = rest % n_seg, o = rest / n_seg;
    const int64_t b = seg ? seg[s] : 0, e = seg ? seg[s + 1] : n;
    const T* p = v + (o * n + b) * inner + k;
    T acc = p[0];
    for (int64_t x = 1; x < e - b; ++x) acc = np_min(acc, p[x * inner]);
    out[t] = acc;
  }
}

template <class T>
int segmin_launch(const void* v, int64_t outer, int64_t n, int64_t inner, const int64_t* seg, int64_t n_seg,
                  void* out, cudaStream_t st) {
  const int64_t total = outer * n_seg * inner;
  if (total == 0) return LCRW_OK;
  segmin_kernel<T><<<grid_for(total), 256, 0, st>>>(static_cast<const T*>(v), outer, n, inner, seg, n_seg,
                                                   static_cast<T*>(out));
  LCRW_CHECK_LAUNCH("segmin_kernel");
  return LCRW_OK;
}

}  // namespace prims
}  // namespace lcrw

using namespace lcrw;

extern "C" {

int lcrw_squared_norms(const void* a, int dtype, int64_t rows, int64_t m, double* out, void* stream) {
  LCRW_REQUIRE(rows >= 0 && m >= 0, "lcrw_squared_norms: bad shape");
  LCRW_REQUIRE(dtype == LCRW_F32 || dtype == LCRW_F64, "lcrw_squared_norms: f32 or f64 rows");
  if (rows == 0) return LCRW_OK;
  LCRW_REQUIRE(out && (a || m == 0), "lcrw_squared_norms: null pointer");
  cudaStream_t st = as_stream(stream);
  if (dtype == LCRW_F32)
    prims::squared_norms_kernel<<<prims::grid_for(rows), 256, 0, st>>>(static_cast<const float*>(a), rows, m, out);
  else
    prims::squared_norms64_kernel<<<prims::grid_for(rows), 256, 0, st>>>(static_cast<const double*>(a), rows, m, out);
  LCRW_CHECK_LAUNCH("squared_norms_kernel");
  return LCRW_OK;
}

int lcrw_euclidean_f64(const double* a, const double* sq_a, int64_t r, const double* b, const double* sq_b, int64_t c,
                       int64_t m, void* out, int out_dtype, int64_t ld, void* stream) {
  LCRW_REQUIRE(out_dtype == LCRW_F32 || out_dtype == LCRW_F64, "lcrw_euclidean_f64: out must be f32 or f64");
  LCRW_REQUIRE(r >= 0 && c >= 0 && m >= 0 && ld >= c, "lcrw_euclidean_f64: bad shape");
  if (r == 0 || c == 0) return LCRW_OK;
  LCRW_REQUIRE(sq_a && sq_b && out && ((a && b) || m == 0), "lcrw_euclidean_f64: null pointer");
  LCRW_REQUIRE(r < 65536 * 1024ll, "lcrw_euclidean_f64: too many rows");
  cudaStream_t st = as_stream(stream);
  const unsigned gx = (unsigned)ceil_div(c, 256);
  for (int64_t r0 = 0; r0 < r; r0 += 65535) {
    const int64_t rr = r - r0 < 65535 ? r - r0 : 65535;
    void* o = static_cast<char*>(out) + (size_t)r0 * ld * (out_dtype == LCRW_F64 ? 8 : 4);
    prims::euclidean_kernel<<<dim3(gx, (unsigned)rr), 256, 0, st>>>(a + r0 * m, sq_a + r0, rr, b, sq_b, c, m, o, ld,
                                                                    out_dtype == LCRW_F64);
    LCRW_CHECK_LAUNCH("euclidean_kernel");
  }
  return LCRW_OK;
}

int lcrw_segmented_min(const void* v, int dtype, int64_t outer, int64_t n, int64_t inner, const int64_t* seg_offsets,
                       int64_t n_seg, void* out, void* stream) {
  LCRW_REQUIRE(outer >= 0 && n >= 1 && inner >= 0 && n_seg >= 1, "lcrw_segmented_min: bad shape");
  LCRW_REQUIRE(v && out, "lcrw_segmented_min: null pointer");
  cudaStream_t st = as_stream(stream);
  switch (dtype) {
    case LCRW_F32: return prims::segmin_launch<float>(v, outer, n, inner, seg_offsets, n_seg, out, st);
    case LCRW_F64: return prims::segmin_launch<double>(v, outer, n, inner, seg_offsets, n_seg, out, st);
    case LCRW_I8: return prims::segmin_launch<int8_t>(v, outer, n, inner, seg_offsets, n_seg, out, st);
    case LCRW_I16: return prims::segmin_launch<int16_t>(v, outer, n, inner, seg_offsets, n_seg, out, st);
    case LCRW_I32: return prims::segmin_launch<int32_t>(v, outer, n, inner, seg_offsets, n_seg, out, st);
    case LCRW_I64: return prims::segmin_launch<int64_t>(v, outer, n, inner, seg_offsets, n_seg, out, st);
    case LCRW_U8: return prims::segmin_launch<uint8_t>(v, outer, n, inner, seg_offsets, n_seg, out, st);
    case LCRW_U16: return prims::segmin_launch<uint16_t>(v, outer, n, inner, seg_offsets, n_seg, out, st);
    case LCRW_U32: return prims::segmin_launch<uint32_t>(v, outer, n, inner, seg_offsets, n_seg, out, st);
    case LCRW_U64: return prims::segmin_launch<uint64_t>(v, outer, n, inner, seg_offsets, n_seg, out, st);
    default: break;
  }
  set_error("lcrw_segmented_min: unsupported dtype code %d", dtype);
  return LCRW_ERR_INVALID;
}

}  // extern "C"
