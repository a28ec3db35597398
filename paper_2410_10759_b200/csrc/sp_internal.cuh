// Internal helpers shared by the splitplan-b200 CUDA translation units.
//
// Nothing here is part of the C ABI (see include/splitplan_b200.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#include "../../include/splitplan_b200.h"

namespace sp {

// ---------------------------------------------------------------------------
// error reporting (sp_abi.cu)

void set_error(int code, const char* fmt, ...);
int check_cuda(cudaError_t err, const char* what);
void set_required_workspace(size_t bytes);
void set_full_workspace(size_t bytes);
void set_steps_overflow(int64_t n);  // instances the last sp_plan_dp re-solved densely
int launch_check(const char* what);  // also counts the launch when profiling

// profiling (sp_abi.cu): events around DP-stage launches
bool profiling();
void prof_record_dp(cudaEvent_t start, cudaEvent_t stop, double cells, double bytes, int variant);

// ---------------------------------------------------------------------------
// IEEE round-to-nearest arithmetic that the compiler may never contract into
// an FMA (the reference evaluates every expression left to right in Python).

__host__ __device__ inline double dadd(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
__host__ __device__ inline double dmul(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
__host__ __device__ inline double ddiv(double a, double b) {
#ifdef __CUDA_ARCH__
  return __ddiv_rn(a, b);
#else
  return a / b;
#endif
}

// ---------------------------------------------------------------------------
// numpy-order floating point reductions
//
// numpy's add.reduce over a contiguous float64 array computes
//   0.0 + pairwise(a, n)
// where pairwise() sums blocks of <= 128 elements with 8 interleaved
// accumulators and splits larger ranges at n/2 rounded down to a multiple of
// 8 (numpy/_core/src/umath/loops_utils.h.src, `DOUBLE_pairwise_sum`).  The
// reference reports every float through np.sum / np.mean
// (planner.py:90-91, evaluator.py:69, throughput_sim.py:122-130), so the
// engine replays the same association order.  `get(i)` yields element i.

// one leaf block (n <= 128)
template <typename Get>
__host__ __device__ inline double pairwise_leaf(const Get& get, int64_t lo, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res = dadd(res, get(lo + i));
    return res;
  }
  double acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = get(lo + j);
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = dadd(acc[j], get(lo + i + j));
  }
  double res = dadd(dadd(dadd(acc[0], acc[1]), dadd(acc[2], acc[3])),
                    dadd(dadd(acc[4], acc[5]), dadd(acc[6], acc[7])));
  for (; i < n; ++i) res = dadd(res, get(lo + i));
  return res;
}

__host__ __device__ inline int64_t pairwise_split(int64_t n) {
  int64_t n2 = n / 2;
  return n2 - n2 % 8;
}

// The recursion pw(a, n) = pw(a, n2) + pw(a + n2, n - n2) for n > 128, run
// with an explicit stack (device threads have a 1 KB default stack; depth is
// at most 64 levels since every level halves n).
template <typename Get>
__host__ __device__ inline double pairwise_sum(const Get& get, int64_t lo0, int64_t n0) {
  if (n0 <= 128) return pairwise_leaf(get, lo0, n0);
  int64_t lo[64], nn[64];
  double left[64];
  uint8_t state[64];  // 1: left child pending, 2: right child pending
  int sp = 0;
  lo[0] = lo0;
  nn[0] = n0;
  state[0] = 0;
  double ret = 0.0;
  while (sp >= 0) {
    if (nn[sp] > 128 && state[sp] == 0) {
      state[sp] = 1;
      lo[sp + 1] = lo[sp];
      nn[sp + 1] = pairwise_split(nn[sp]);
      state[sp + 1] = 0;
      ++sp;
      continue;
    }
    ret = pairwise_leaf(get, lo[sp], nn[sp]);
    --sp;
    while (sp >= 0) {  // hand the finished subtree to its parents
      if (state[sp] == 1) {
        left[sp] = ret;
        state[sp] = 2;
        const int64_t n2 = pairwise_split(nn[sp]);
        lo[sp + 1] = lo[sp] + n2;
        nn[sp + 1] = nn[sp] - n2;
        state[sp + 1] = 0;
        ++sp;
        break;
      }
      ret = dadd(left[sp], ret);
      --sp;
    }
  }
  return ret;
}

template <typename Get>
__host__ __device__ inline double np_sum(const Get& get, int64_t n) {
  return dadd(0.0, pairwise_sum(get, 0, n));
}

// ---------------------------------------------------------------------------
// value modes of the DP tables

enum ValueMode : int32_t {
  VM_INT32 = 0,    // all r integral, sum(r) < 2^53, sum(r)/g < 2^31: exact int32 DP
  VM_F64 = 1,      // all r finite: fp64 DP, tables never hold NaN
  VM_F64_NAN = 2,  // some r non-finite: fp64 DP with numpy NaN propagation
};

// per-instance record written by the prep kernel
struct InstInfo {
  int64_t w_eff;     // planner.py:120-125
  double scale;      // g: r_k = g * rv_k in VM_INT32
  double end_c;      // C[L][W_eff]
  double end_s;      // S[L][W_eff]
  int32_t mode;      // ValueMode
  int32_t pad;
};

// per-layer stage record, shifts clamped to W_eff + 1 (a shift beyond the
// row leaves every cell unreachable, planner.py:110-117)
struct StageShift {
  int32_t i;    // client compute
  int32_t id;   // i + d (switch server -> client)
  int32_t s;    // server compute
  int32_t su;   // s + u (switch client -> server)
};

// work item of one DP CTA
struct DpWork {
  int64_t inst;
  int64_t bp_off;        // byte offset of this instance's back-pointer table
  int64_t row_off;       // byte offset of its global rows, or -1 if rows live in SMEM
  int64_t bp_row_words;  // u32 words per stage row of the back-pointer table
};

}  // namespace sp
