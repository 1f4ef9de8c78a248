// Host-side plumbing of the C ABI: thread-local error strings, launch checks, launch counter.
#include <cstdarg>
#include <cstdio>
#include <atomic>

#include "pf_common.cuh"

namespace pf {

static thread_local char g_err[1024] = "";
static std::atomic<uint64_t> g_launches{0};

int set_error(int status, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return status;
}

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int check_launch(const char* what) {
  note_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(PF_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return PF_OK;
}

}  // namespace pf

extern "C" {

const char* pf_last_error(void) { return pf::g_err; }
int pf_abi_version(void) { return PF_ABI_VERSION; }
uint64_t pf_launch_count(void) { return pf::g_launches.load(); }

}  // extern "C"
