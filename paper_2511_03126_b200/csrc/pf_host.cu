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

// ---- stage timer: CUDA events at the stage boundaries of the fused tile path -------------------------
// Mark m of call c is event g_ev[c % kRing][m]; pf_stage_times sums the intervals over the calls
// recorded since pf_stage_timing(1). Events are recorded on the launching stream.
constexpr int kRing = 64;
static bool g_timing = false;
static cudaEvent_t g_ev[kRing][kStageMarks];
static bool g_ev_made = false;
static int g_calls = 0;
static int g_marks_seen[kRing];

void stage_mark(int mark, cudaStream_t st) {
  if (!g_timing || mark < 0 || mark >= kStageMarks) return;
  if (mark == 0) {
    ++g_calls;
    g_marks_seen[(g_calls - 1) % kRing] = 0;
  }
  if (g_calls == 0) return;
  const int c = (g_calls - 1) % kRing;
  cudaEventRecord(g_ev[c][mark], st);
  g_marks_seen[c] |= 1 << mark;
}

}  // namespace pf

extern "C" {

int pf_stage_timing(int enable) {
  using namespace pf;
  if (enable && !g_ev_made) {
    for (auto& row : g_ev)
      for (auto& e : row)
        if (cudaEventCreate(&e) != cudaSuccess) return set_error(PF_ERR_CUDA, "stage_timing: event create");
    g_ev_made = true;
  }
  g_timing = enable != 0;
  g_calls = 0;
  return PF_OK;
}

int pf_stage_times(float* ms, int32_t n) {
  using namespace pf;
  if (!ms || n < 1) return -set_error(PF_ERR_VALUE, "stage_times: need an output array");
  for (int q = 0; q < n; ++q) ms[q] = 0.f;
  const int calls = g_calls < kRing ? g_calls : kRing;
  for (int c = 0; c < calls; ++c) {
    int prev = -1;
    for (int m = 0; m < kStageMarks; ++m) {
      if (!(g_marks_seen[c] & (1 << m))) continue;
      if (prev >= 0 && m - 1 < n) {
        float t = 0.f;
        if (cudaEventSynchronize(g_ev[c][m]) != cudaSuccess ||
            cudaEventElapsedTime(&t, g_ev[c][prev], g_ev[c][m]) != cudaSuccess)
          return -set_error(PF_ERR_CUDA, "stage_times: %s", cudaGetErrorString(cudaGetLastError()));
        ms[m - 1] += t;
      }
      prev = m;
    }
  }
  return calls;
}

const char* pf_last_error(void) { return pf::g_err; }
int pf_abi_version(void) { return PF_ABI_VERSION; }
uint64_t pf_launch_count(void) { return pf::g_launches.load(); }

}  // extern "C"
