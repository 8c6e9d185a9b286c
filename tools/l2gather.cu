// L2 gather ceiling probe (the "peak" of bench.py's table_min roofline, profiles/l2_gather_peak.json):
// 512-byte (32 lanes x 16 B, the current table row) and 480-byte random row gathers + min
// from an L2-resident ~50 MB table, the access pattern of csrc/table.cu without its Z2 stores.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/l2gather tools/l2gather.cu
// Microbenchmark: random 512-B (or 1-KB) row gathers + min from an L2-resident table,
// the access pattern of a distance-table formulation of the reverse Phase 1.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>
#include <random>

__global__ void fill(float* t, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    t[i] = (float)((i * 2654435761u) % 1000003u) * 1e-3f;
}

template <int VEC>  // float4 per lane per row: row width = 32*4*VEC floats (lanes < act_lanes load)
__global__ void __launch_bounds__(256) gather_min(const float4* __restrict__ T, int row_f4, const int* __restrict__ cols,
                                                  int h, int n_docs, float4* __restrict__ out, int act_lanes) {
  const int lane = threadIdx.x & 31;
  const bool act = lane < act_lanes;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int d = warp; d < n_docs; d += nw) {
    const int* c = cols + (int64_t)d * h;
    int myc = lane < h ? __ldg(c + lane) : 0;
    int myc2 = lane + 32 < h ? __ldg(c + 32 + lane) : 0;
    float4 acc[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[v] = make_float4(3e38f, 3e38f, 3e38f, 3e38f);
#pragma unroll 8
    for (int j = 0; j < h; ++j) {
      const int u = __shfl_sync(0xffffffffu, j < 32 ? myc : myc2, j & 31);
      const float4* r = T + (int64_t)u * row_f4 + lane;
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        if (!act) continue;
        float4 x = __ldg(r + 32 * v);
        acc[v].x = fminf(acc[v].x, x.x); acc[v].y = fminf(acc[v].y, x.y);
        acc[v].z = fminf(acc[v].z, x.z); acc[v].w = fminf(acc[v].w, x.w);
      }
    }
#pragma unroll
    for (int v = 0; v < VEC; ++v) if (act) out[((int64_t)(d & 4095) * VEC + v) * 32 + lane] = acc[v];
  }
}

// the table_min access pattern at its best: word ids broadcast four at a time from a per-warp
// smem slot (LDS.128) instead of a SHFL per row, no predication (lanes past act_lanes re-read
// the last active lane's 16 bytes), 8 rows in flight per warp
__global__ void __launch_bounds__(256) gather_min_q(const uint4* __restrict__ T, int row_f4, const int* __restrict__ cols,
                                                    int h, int n_docs, uint4* __restrict__ out, int act_lanes) {
  __shared__ __align__(16) int ids[8][64];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int my = lane < act_lanes ? lane : act_lanes - 1;
  for (int d = warp; d < n_docs; d += nw) {
    const int* c = cols + (int64_t)d * h;
    __syncwarp();
    ids[wl][lane] = lane < h ? __ldg(c + lane) : 0;
    ids[wl][lane + 32] = lane + 32 < h ? __ldg(c + 32 + lane) : 0;
    __syncwarp();
    uint4 acc = make_uint4(~0u, ~0u, ~0u, ~0u);
    const int4* q4 = reinterpret_cast<const int4*>(ids[wl]);
    int j = 0;
#pragma unroll 2
    for (; j + 4 <= h; j += 4) {
      const int4 u = q4[j >> 2];
      const uint4 a = __ldg(T + (int64_t)u.x * row_f4 + my), b = __ldg(T + (int64_t)u.y * row_f4 + my);
      const uint4 e = __ldg(T + (int64_t)u.z * row_f4 + my), f = __ldg(T + (int64_t)u.w * row_f4 + my);
      acc.x = min(min(acc.x, a.x), min(b.x, min(e.x, f.x)));
      acc.y = min(min(acc.y, a.y), min(b.y, min(e.y, f.y)));
      acc.z = min(min(acc.z, a.z), min(b.z, min(e.z, f.z)));
      acc.w = min(min(acc.w, a.w), min(b.w, min(e.w, f.w)));
    }
    for (; j < h; ++j) {
      const uint4 a = __ldg(T + (int64_t)ids[wl][j] * row_f4 + my);
      acc.x = min(acc.x, a.x); acc.y = min(acc.y, a.y); acc.z = min(acc.z, a.z); acc.w = min(acc.w, a.w);
    }
    if (lane < act_lanes) out[(int64_t)(d & 4095) * 32 + lane] = acc;
  }
}

int main() {
  const int V = 100000, h = 50, n_docs = 1000000;
  std::vector<int> hc((size_t)n_docs * h);
  std::mt19937 g(1);
  for (auto& x : hc) x = g() % V;
  int* cols; cudaMalloc(&cols, hc.size() * 4); cudaMemcpy(cols, hc.data(), hc.size() * 4, cudaMemcpyHostToDevice);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int act_lanes : {30, 32}) {
    const int row_f4 = act_lanes;
    float4* T; cudaMalloc(&T, (size_t)V * row_f4 * 16);
    fill<<<4096, 256>>>(reinterpret_cast<float*>(T), (int64_t)V * row_f4 * 4);
    float4* out; cudaMalloc(&out, (size_t)4096 * 32 * 16);
    for (int bps : {4, 8, 16, 64}) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      auto run = [&]() {
        gather_min<1><<<sms * bps, 256>>>(T, row_f4, cols, h, n_docs, out, act_lanes);
      };
      run(); run();
      cudaEventRecord(a);
      for (int i = 0; i < 10; ++i) run();
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
      double bytes = (double)n_docs * h * row_f4 * 16;
      printf("row %d B table %.1f MB blocks/SM %d: %.3f ms  %.2f TB/s gathered  err=%s\n", row_f4 * 16,
             V * row_f4 * 16 / 1e6, bps, ms, bytes / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    for (int bps : {4, 8, 16, 64}) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      auto run = [&]() {
        gather_min_q<<<sms * bps, 256>>>(reinterpret_cast<const uint4*>(T), row_f4, cols, h, n_docs,
                                         reinterpret_cast<uint4*>(out), act_lanes);
      };
      run(); run();
      cudaEventRecord(a);
      for (int i = 0; i < 10; ++i) run();
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
      double bytes = (double)n_docs * h * row_f4 * 16;
      printf("row %d B table %.1f MB blocks/SM %d smem-quad ids: %.3f ms  %.2f TB/s gathered  err=%s\n", row_f4 * 16,
             V * row_f4 * 16 / 1e6, bps, ms, bytes / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    cudaFree(T); cudaFree(out);
  }
  return 0;
}
