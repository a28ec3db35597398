// Library-level state of the C ABI: thread-local error text, status helpers.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include "sp_internal.cuh"

#include <vector>

namespace {
thread_local char g_err[1024] = "";
thread_local size_t g_required_ws = 0;
thread_local size_t g_full_ws = 0;
thread_local int64_t g_steps_overflow = 0;

struct DpRec {
  cudaEvent_t a, b;
  double cells, bytes;
  int variant;
};
thread_local bool g_prof = false;
thread_local int64_t g_launches = 0;
thread_local std::vector<DpRec> g_dp;
}  // namespace

namespace sp {

void set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  int n = snprintf(g_err, sizeof(g_err), "[sp status %d] ", code);
  if (n < 0) n = 0;
  vsnprintf(g_err + n, sizeof(g_err) - (size_t)n, fmt, ap);
  va_end(ap);
}

int check_cuda(cudaError_t err, const char* what) {
  if (err == cudaSuccess) return SP_OK;
  set_error(SP_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorString(err), cudaGetErrorName(err));
  return SP_ERR_CUDA;
}

int launch_check(const char* what) {
  if (g_prof) ++g_launches;
  return check_cuda(cudaGetLastError(), what);
}

void set_required_workspace(size_t bytes) { g_required_ws = bytes; }
void set_full_workspace(size_t bytes) { g_full_ws = bytes; }
void set_steps_overflow(int64_t n) { g_steps_overflow = n; }

bool profiling() { return g_prof; }

void prof_record_dp(cudaEvent_t start, cudaEvent_t stop, double cells, double bytes, int variant) {
  g_dp.push_back(DpRec{start, stop, cells, bytes, variant});
}

}  // namespace sp

extern "C" {

void sp_profile_enable(int on) { g_prof = on != 0; }

int sp_profile_collect(double* dp_kernel_ms, int64_t* dp_launches, double* dp_cells,
                       double* dp_bytes, int64_t* all_launches, int32_t* dp_variant) {
  double ms = 0, cells = 0, bytes = 0;
  double by_variant[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int rc = SP_OK;
  for (DpRec& r : g_dp) {
    float t = 0.f;
    if (rc == SP_OK) rc = sp::check_cuda(cudaEventSynchronize(r.b), "profile event sync");
    if (rc == SP_OK) rc = sp::check_cuda(cudaEventElapsedTime(&t, r.a, r.b), "profile elapsed");
    ms += t;
    if (r.variant >= 0 && r.variant < 8) by_variant[r.variant] += t;
    cells += r.cells;
    bytes += r.bytes;
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  if (dp_kernel_ms) *dp_kernel_ms = ms;
  if (dp_launches) *dp_launches = (int64_t)g_dp.size();
  if (dp_cells) *dp_cells = cells;
  if (dp_bytes) *dp_bytes = bytes;
  if (all_launches) *all_launches = g_launches;
  if (dp_variant) {
    int best = 0;
    for (int v = 1; v < 8; ++v)
      if (by_variant[v] > by_variant[best]) best = v;
    *dp_variant = best;
  }
  g_dp.clear();
  g_launches = 0;
  return rc;
}

int sp_abi_version(void) { return SP_ABI_VERSION; }

const char* sp_last_error(void) { return g_err; }

size_t sp_last_required_workspace(void) { return g_required_ws; }

size_t sp_last_full_workspace(void) { return g_full_ws; }

int64_t sp_last_dense_fallbacks(void) { return g_steps_overflow; }

}  // extern "C"
