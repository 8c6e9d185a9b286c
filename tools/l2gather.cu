// L2 gather ceiling probe (the "peak" of bench.py's table_min roofline, profiles/l2_gather_peak.json):
// 480-byte (30 lanes x 16 B, the current table row) and 512-byte random row gathers + min
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
    cudaFree(T); cudaFree(out);
  }
  return 0;
}
