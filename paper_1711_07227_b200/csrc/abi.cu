// C-ABI plumbing: status strings, thread-local error messages, device facts.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

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

// ---------------------------------------------------------------------------
// optional launch profiler: CUDA events around instrumented launches on the
// launching stream (bench.py enables it to time kernels inside the timed
// region without host synchronisation; read back after a synchronize).
// ---------------------------------------------------------------------------
namespace {
struct ProfRec {
  char name[32];
  cudaEvent_t a, b;
};
std::mutex g_mu;
bool g_prof = false;
std::vector<ProfRec> g_recs;
std::vector<cudaEvent_t> g_pool;
size_t g_pool_used = 0;

cudaEvent_t pool_event() {
  if (g_pool_used == g_pool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    g_pool.push_back(e);
  }
  return g_pool[g_pool_used++];
}
}  // namespace

ProfScope::ProfScope(cudaStream_t s, const char* name) : stream_(s), name_(name), a_(nullptr) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_prof) return;
  a_ = pool_event();
  if (a_) cudaEventRecord(a_, s);
}

ProfScope::~ProfScope() {
  if (!a_) return;
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_prof) return;
  cudaEvent_t b = pool_event();
  if (!b) return;
  cudaEventRecord(b, stream_);
  ProfRec r;
  std::strncpy(r.name, name_, sizeof(r.name) - 1);
  r.name[sizeof(r.name) - 1] = 0;
  r.a = a_;
  r.b = b;
  g_recs.push_back(r);
}

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

int lcrw_operand_k(int m, int split) { return m <= 0 ? 0 : (split ? 3 * m : m) + 3; }

int lcrw_profile_reset(int enable) {
  std::lock_guard<std::mutex> lk(lcrw::g_mu);
  lcrw::g_recs.clear();
  lcrw::g_pool_used = 0;
  lcrw::g_prof = enable != 0;
  return LCRW_OK;
}

int64_t lcrw_profile_count(void) {
  std::lock_guard<std::mutex> lk(lcrw::g_mu);
  return (int64_t)lcrw::g_recs.size();
}

int lcrw_profile_get(int64_t i, char* name, int name_cap, float* ms) {
  std::lock_guard<std::mutex> lk(lcrw::g_mu);
  if (i < 0 || i >= (int64_t)lcrw::g_recs.size() || !name || name_cap < 2 || !ms) return LCRW_ERR_INVALID;
  const auto& r = lcrw::g_recs[(size_t)i];
  std::strncpy(name, r.name, (size_t)name_cap - 1);
  name[name_cap - 1] = 0;
  cudaError_t e = cudaEventSynchronize(r.b);
  if (e != cudaSuccess) return lcrw::cuda_status(e, "cudaEventSynchronize (profile)");
  e = cudaEventElapsedTime(ms, r.a, r.b);
  if (e != cudaSuccess) return lcrw::cuda_status(e, "cudaEventElapsedTime (profile)");
  return LCRW_OK;
}

}  // extern "C"
