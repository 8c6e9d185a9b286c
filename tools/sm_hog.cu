// Probe (not shipped): occupy n SMs with spinning CTAs that hold ~200 KB of shared memory
// each, so a concurrently running kernel gets the remaining SMs only.  Used by
// tools/sm_share.py to ask whether table_min keeps its rate on fewer SMs (L2-bound) or
// slows in proportion (SM-bound) -- the premise of overlapping it with the reverse SpMM.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o tools/libsmhog.so tools/sm_hog.cu
#include <cstdint>
#include <cuda_runtime.h>

__global__ void hog_kernel(volatile int* stop) {
  extern __shared__ int s[];
  if (threadIdx.x == 0) {
    s[0] = 0;
    while (*stop == 0) __nanosleep(1000);
  }
}

extern "C" int sm_hog_launch(int n_ctas, int* stop, void* stream) {
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(hog_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  hog_kernel<<<n_ctas, 32, smem, static_cast<cudaStream_t>(stream)>>>(stop);
  return (int)cudaGetLastError();
}
