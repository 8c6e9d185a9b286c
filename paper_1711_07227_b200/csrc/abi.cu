// C-ABI plumbing: status strings, thread-local error messages, device facts.
#include <cstdarg>
#include <cstdio>

#include "common.cuh"

namespace lcrw {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char* what) {
  set_error("%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
  return LCRW_ERR_CUDA;
}

int sm_count() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) return 148;
  return n;
}

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace lcrw

extern "C" {

int lcrw_abi_version(void) { return 1; }

const char* lcrw_status_string(int status) {
  switch (status) {
    case LCRW_OK: return "ok";
    case LCRW_ERR_INVALID: return "invalid argument";
    case LCRW_ERR_CUDA: return "CUDA error";
    case LCRW_ERR_UNSUPPORTED: return "unsupported shape";
    default: return "unknown status";
  }
}

const char* lcrw_last_error(void) { return lcrw::g_err; }

int lcrw_sm_count(int* out) {
  if (!out) return LCRW_ERR_INVALID;
  *out = lcrw::sm_count();
  return LCRW_OK;
}

int lcrw_padded_dim(int m) { return m <= 0 ? 0 : ((m + 63) / 64) * 64; }

}  // extern "C"
