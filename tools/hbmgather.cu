// Probe for a gather form of the reverse SpMM: warps read 128-byte Z2 rows
// (32 docs x f32 of one word) of 5-MB panels in the order of query word lists, panels
// taken in sequence by all warps (p-major work items from an atomic counter), so each
// panel is fetched from HBM about once and re-read from L2 for the words several queries
// share.  Reports the panel bytes streamed per second (the HBM-side rate).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/hbmgather tools/hbmgather.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>

__device__ unsigned long long g_next;

__global__ void __launch_bounds__(256) gather_rows(const float* __restrict__ Z, int64_t rows, int64_t n_panels,
                                                    const int* __restrict__ q_off, const int* __restrict__ q_rows,
                                                    int n_q, int qpi, float* __restrict__ out, int prefetch) {
  const int lane = threadIdx.x & 31;
  const int64_t items_per_panel = (n_q + qpi - 1) / qpi;
  const int64_t n_items = n_panels * items_per_panel;
  for (;;) {
    unsigned long long it = 0;
    if (lane == 0) it = atomicAdd(&g_next, 1ull);
    it = __shfl_sync(0xffffffffu, it, 0);
    if ((int64_t)it >= n_items) break;
    const int64_t p = it / items_per_panel, b = it - p * items_per_panel;
    const float* zp = Z + p * rows * 32;
    if (prefetch && b == 0 && lane == 0 && p + 2 < n_panels)  // stream a panel ahead into L2
      for (int64_t off = 0; off < rows * 128; off += 65536) {
        const uint32_t bytes = (uint32_t)min((int64_t)65536, rows * 128 - off);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<const char*>(Z + (p + 2) * rows * 32) + off), "r"(bytes) : "memory");
      }
    float sum = 0.f;
    for (int q = (int)(b * qpi); q < min(n_q, (int)((b + 1) * qpi)); ++q) {
      float acc = 0.f;
      const int e = q_off[q + 1];
      int j = q_off[q];
#pragma unroll 1
      for (; j + 8 <= e; j += 8) {
        float z[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) z[u] = __ldg(zp + (int64_t)__ldg(q_rows + j + u) * 32 + lane);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = fmaf(0.5f, z[u], acc);
      }
      for (; j < e; ++j) acc = fmaf(0.5f, __ldg(zp + (int64_t)__ldg(q_rows + j) * 32 + lane), acc);
      sum += acc;
    }
    if (sum == -1.f) out[lane] = sum;
  }
}

int main() {
  const int64_t rows = 39400, n_panels = 3000;  // 3000 x 5 MB = 15 GB of Z2
  const int n_q = 1000, h = 50;
  std::mt19937 g(1);
  std::vector<int> off(n_q + 1), qr;
  for (int q = 0; q < n_q; ++q) {
    std::vector<int> w(h);
    for (auto& x : w) x = (int)(g() % rows);
    std::sort(w.begin(), w.end());
    qr.insert(qr.end(), w.begin(), w.end());
    off[q + 1] = (int)qr.size();
  }
  float* Z; cudaMalloc(&Z, (size_t)rows * 32 * 4 * n_panels);
  cudaMemset(Z, 0, (size_t)rows * 32 * 4 * n_panels);
  int *d_off, *d_rows; float* out;
  cudaMalloc(&d_off, off.size() * 4); cudaMalloc(&d_rows, qr.size() * 4); cudaMalloc(&out, 128);
  cudaMemcpy(d_off, off.data(), off.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_rows, qr.data(), qr.size() * 4, cudaMemcpyHostToDevice);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int prefetch : {0, 1})
    for (int qpi : {1, 2, 8})
      for (int bps : {4, 8}) {
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        unsigned long long zero = 0;
        auto run = [&]() {
          cudaMemcpyToSymbol(g_next, &zero, 8);
          gather_rows<<<sms * bps, 256>>>(Z, rows, n_panels, d_off, d_rows, n_q, qpi, out, prefetch);
        };
        run();
        cudaEventRecord(a);
        run();
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        const double panel_bytes = (double)rows * 128 * n_panels;
        printf("prefetch %d queries/item %d blocks/SM %d: %.2f ms  panels %.2f TB/s  gathers %.2f TB/s  err=%s\n",
               prefetch, qpi, bps, ms, panel_bytes / ms / 1e9, (double)qr.size() * 128 * n_panels / ms / 1e9,
               cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
