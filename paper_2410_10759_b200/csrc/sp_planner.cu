// Planner kernels of the B200 placement engine (reference: planner.py).
//
//   dp_core.cuh        prep_kernel (W_eff, value domain, clamped stage shifts,
//                      reachable frontiers), the per-cell update, and
//                      dp_stage_kernel: K2 with rows in one CTA's SMEM
//                      (planner.py:128-143), 2-bit packed back-pointers
//   dp_stream.cuh      K2 for wide rows: dp_stream_kernel (L2 rows, bulk-copy
//                      windows)
//   dp_grid.cuh        K2 for one huge instance (cfg5): dp_grid_kernel over
//                      capacity partitions, checkpoint/backtrack kernels
//   dp_steps.cuh       K2 + K3 on breakpoint lists (rows as step functions):
//                      dp_steps_kernel (forward pass, walk back, _finish)
//   this file          backtrack_kernel (K3: end-side choice + pointer walk +
//                      _finish, planner.py:88-107, 146-202), prefix_kernel
//                      (greedy / all-server / all-client, planner.py:205-225),
//                      exhaustive_kernel (plan_oracle, planner.py:228-268),
//                      eq1_kernel (latency_of, evaluator.py:64-78), the host
//                      planning of waves / variants / geometry, and the C ABI.
//
// See DESIGN.md for the data layout and the value domains.
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <type_traits>
#include <vector>

#include "sp_internal.cuh"

namespace sp {
namespace {

constexpr int kStageTile = 128;          // stage records staged in SMEM at a time
constexpr size_t kSmemCap = 227 * 1024;  // sm_100a max dynamic SMEM per CTA
constexpr int64_t kMaxCols = (int64_t(1) << 31) - 64;
constexpr int64_t kGridMinColsSteps = (int64_t)1 << 22;  // == kGridMinCols: whole-GPU widths stay dense

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

#include "dp_core.cuh"
#include "dp_stream.cuh"
#include "dp_grid.cuh"
#include "dp_steps.cuh"

// ---------------------------------------------------------------------------
// _finish over caller-supplied placements

__global__ void evaluate_kernel(sp_instances in, const uint8_t* pi_in, sp_policies out,
                                int32_t* idx_scratch) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= in.n) return;
  const int64_t lo = in.layer_off[t];
  const int L = (int)(in.layer_off[t + 1] - lo);
  if (out.pi != pi_in)
    for (int k = 0; k < L; ++k) out.pi[lo + k] = pi_in[lo + k] ? 1 : 0;
  finish_policy(in, t, lo, L, idx_scratch + lo, out, false, false);
  out.status[t] = SP_OK;
}

// ---------------------------------------------------------------------------
// K3: end-side argmax + back-pointer walk + finish (planner.py:146-202)

__global__ void backtrack_kernel(sp_instances in, const InstInfo* info, const StageShift* shifts,
                                 const DpWork* work, int64_t n_work, const uint8_t* bp,
                                 int32_t* idx_scratch, sp_policies out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_work) return;
  const DpWork wk = work[t];
  const int64_t inst = wk.inst;
  const int64_t lo = in.layer_off[inst];
  const int L = (int)(in.layer_off[inst + 1] - lo);
  const InstInfo inf = info[inst];
  double ec = inf.end_c, es = inf.end_s;
  const int8_t must = in.must_end_at ? in.must_end_at[inst] : (int8_t)-1;
  if (must == 1) es = -INFINITY;
  else if (must == 0) ec = -INFINITY;
  const double pmax = (es > ec) ? es : ec;  // Python builtin max(end_c, end_s)
  uint8_t* pi = out.pi + lo;
  int32_t status = SP_OK;
  if (pmax == -INFINITY) {  // _infeasible
    for (int k = 0; k < L; ++k) pi[k] = 0;
    finish_policy(in, inst, lo, L, idx_scratch + lo, out, true, false);
    out.status[inst] = SP_OK;
    return;
  }
  bool client = ec >= es;
  int64_t j = inf.w_eff;
  // packed back-pointer words: per row, per 32-column group, nw words
  // (C-stay, S-stay[, C-switch, S-switch]); see the K2 comment
  const uint32_t* bpi = reinterpret_cast<const uint32_t*>(bp + wk.bp_off);
  const int nw = bp_words(inf.mode);
  const int64_t row_words = wk.bp_row_words;
  for (int k = L; k >= 1; --k) {
    const uint32_t* grp = bpi + (int64_t)(k - 1) * row_words + (j >> 5) * nw;
    const uint32_t bit = 1u << (j & 31);
    const bool c_stay = grp[0] & bit, s_stay = grp[1] & bit;
    const bool c_sw = nw == 4 ? (grp[2] & bit) != 0 : !c_stay;
    const bool s_sw = nw == 4 ? (grp[3] & bit) != 0 : !s_stay;
    const uint32_t b = (c_stay ? 1u : 0u) | (c_sw ? 2u : 0u) | (s_stay ? 4u : 0u) | (s_sw ? 8u : 0u);
    const StageShift sh = shifts[lo + k - 1];
    if (client) {
      pi[k - 1] = 1;
      if (b & 1u) {
        j -= sh.i;
      } else if (b & 2u) {
        j -= sh.id;
        client = false;
      } else {
        status = SP_ERR_BACKTRACE;
        break;
      }
    } else {
      pi[k - 1] = 0;
      if (b & 4u) {
        j -= sh.s;
      } else if (b & 8u) {
        j -= sh.su;
        client = true;
      } else {
        status = SP_ERR_BACKTRACE;
        break;
      }
    }
  }
  out.status[inst] = status;
  if (status != SP_OK) return;
  finish_policy(in, inst, lo, L, idx_scratch + lo, out, false, false);
}

// ---------------------------------------------------------------------------
// prefix planners: one warp per instance, warp-scan over split points m

__global__ void prefix_kernel(sp_instances in, int32_t which, sp_policies out) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= in.n) return;
  const int64_t lo = in.layer_off[w];
  const int64_t L = in.layer_off[w + 1] - lo;
  const bool sac = in.source_at_client[w] != 0;
  const int64_t budget = in.budget[w];
  const int64_t* I = in.client_units + lo;
  const int64_t* S = in.server_units + lo;
  const int64_t* U = in.up_units + lo;
  const int64_t d0 = in.down_units[lo];

  int64_t stot = 0, itot = 0;
  for (int64_t k = lane; k < L; k += 32) {
    stot += S[k];
    itot += I[k];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    stot += __shfl_xor_sync(0xffffffffu, stot, o);
    itot += __shfl_xor_sync(0xffffffffu, itot, o);
  }
  // lat(m) = sum_{k<m} i_k + sum_{k>=m} s_k + [m<L and (m>=1 or sac)] u_m + [m>=1 and !sac] d_0
  auto lat_of = [&](int64_t m, int64_t pre_i, int64_t pre_s) {
    int64_t v = pre_i + (stot - pre_s);
    if (m < L && (m >= 1 || sac)) v += U[m];
    if (m >= 1 && !sac) v += d0;
    return v;
  };
  int64_t m_sel = 0;
  bool ok_sel = false;
  int64_t lat_sel = 0;
  if (which == SP_ALL_SERVER) {
    m_sel = 0;
    lat_sel = lat_of(0, 0, 0);
  } else if (which == SP_ALL_CLIENT) {
    m_sel = L;
    lat_sel = lat_of(L, itot, stot);
  } else {
    int64_t carry_i = 0, carry_s = 0;
    int64_t best = -1, best_lat = 0;
    for (int64_t base = 0; base <= L; base += 32) {
      const int64_t m = base + lane;
      const int64_t own_i = (m < L) ? I[m] : 0;
      const int64_t own_s = (m < L) ? S[m] : 0;
      int64_t inc_i = own_i, inc_s = own_s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t vi = __shfl_up_sync(0xffffffffu, inc_i, o);
        const int64_t vs = __shfl_up_sync(0xffffffffu, inc_s, o);
        if (lane >= o) {
          inc_i += vi;
          inc_s += vs;
        }
      }
      const int64_t pre_i = carry_i + inc_i - own_i;  // sum_{k<m} i_k
      const int64_t pre_s = carry_s + inc_s - own_s;
      const int64_t lm = lat_of(m, pre_i, pre_s);
      const bool ok = (m <= L) && lm <= budget;
      const unsigned ball = __ballot_sync(0xffffffffu, ok);
      if (ball) {
        const int hl = 31 - __clz(ball);
        best = base + hl;
        best_lat = __shfl_sync(0xffffffffu, lm, hl);
      }
      carry_i += __shfl_sync(0xffffffffu, inc_i, 31);
      carry_s += __shfl_sync(0xffffffffu, inc_s, 31);
    }
    if (best >= 0) {
      m_sel = best;
      lat_sel = best_lat;
      ok_sel = true;
    } else {
      m_sel = 0;
      lat_sel = lat_of(0, 0, 0);
    }
  }
  for (int64_t k = lane; k < L; k += 32) out.pi[lo + k] = k < m_sel ? 1 : 0;
  if (lane == 0) {
    const double* r = in.r + lo;
    out.client_value[w] = np_sum([&](int64_t m) { return r[m]; }, m_sel);
    out.server_load[w] = np_sum([&](int64_t m) { return r[m_sel + m]; }, L - m_sel);
    out.integer_latency[w] = lat_sel;
    out.feasible[w] = (which == SP_GREEDY) ? (ok_sel ? 1 : 0) : (lat_sel <= budget ? 1 : 0);
    out.status[w] = SP_OK;
  }
}

// ---------------------------------------------------------------------------
// exhaustive planner (plan_oracle, planner.py:228-268): one CTA per instance

// value = x @ r (planner.py:253) exactly as numpy evaluates it on the host the
// golden vectors come from: numpy hands the (masks x L) @ (L,) product to
// OpenBLAS dgemv_t (0.3.30, the Haswell/SkylakeX micro-kernel), which sums
// the first 4*floor(L/4) layers in four lane-strided accumulators (lane k
// takes layers k, k+4, ... in order; x in {0, 1} makes each FMA an add),
// reduces them as (a0 + a2) + (a1 + a3), then adds the last L mod 4 layers
// summed left to right (a model checked against numpy on 51k masks, 0
// mismatches; profiles/r02/oracle_blas_order.json).  0 * inf = NaN as in BLAS.
__device__ double mask_value(const double* r, int L, uint32_t mask) {
  const int m3 = L & 3, m1 = L - m3;
  auto x = [&](int i) { return ((mask >> (L - 1 - i)) & 1u) ? 1.0 : 0.0; };  // layer 1 is the MSB
  double y = 0.0;
  if (m1) {
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    for (int i = 0; i < m1; ++i) a[i & 3] = dadd(a[i & 3], dmul(x(i), r[i]));
    y = dadd(y, dadd(dadd(a[0], a[2]), dadd(a[1], a[3])));
  }
  if (m3) {
    double t = dmul(x(m1), r[m1]);
    for (int i = m1 + 1; i < L; ++i) t = dadd(t, dmul(x(i), r[i]));
    y = dadd(y, t);
  }
  return y;
}

struct MaskBest {
  double v;
  uint32_t m;
  int found;
};

// np.argmax order inside one chunk of masks: NaN first, then the larger
// value, ties to the smaller mask (the first index)
__device__ __forceinline__ bool mask_better(const MaskBest& a, const MaskBest& b) {
  if (!a.found) return false;
  if (!b.found) return true;
  const bool an = a.v != a.v, bn = b.v != b.v;
  if (an || bn) return an && (!bn || a.m < b.m);
  return a.v > b.v || (a.v == b.v && a.m < b.m);
}

__global__ void exhaustive_kernel(sp_instances in, sp_policies out) {
  constexpr uint32_t kChunk = 1u << 16;  // planner.py:228 default chunk
  const int64_t inst = blockIdx.x;
  const int64_t lo = in.layer_off[inst];
  const int L = (int)(in.layer_off[inst + 1] - lo);
  const bool sac = in.source_at_client[inst] != 0;
  const int64_t budget = in.budget[inst];
  const double* r = in.r + lo;
  __shared__ double s_val[32];
  __shared__ uint32_t s_mask[32];
  __shared__ int s_found[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  MaskBest best{-INFINITY, 0xffffffffu, 0};  // across chunks (thread 0)
  const uint32_t nmask = 1u << L;
  for (uint32_t start = 0; start < nmask; start += kChunk) {
    const uint32_t stop = min(nmask, start + kChunk);
    MaskBest cb{-INFINITY, 0xffffffffu, 0};
    for (uint32_t mask = start + threadIdx.x; mask < stop; mask += blockDim.x) {
      int64_t lat = 0;  // exact: the reference's float np.sum of integral terms (< 2^53)
      int prev = sac ? 1 : 0;
      for (int k = 0; k < L; ++k) {
        const int xk = (mask >> (L - 1 - k)) & 1;
        lat += xk ? in.client_units[lo + k] + (prev ? 0 : in.down_units[lo + k])
                  : in.server_units[lo + k] + (prev ? in.up_units[lo + k] : 0);
        prev = xk;
      }
      if (lat > budget) continue;
      const MaskBest c{mask_value(r, L, mask), mask, 1};
      if (mask_better(c, cb)) cb = c;
    }
    for (int o = 16; o > 0; o >>= 1) {
      MaskBest other;
      other.v = __shfl_xor_sync(0xffffffffu, cb.v, o);
      other.m = __shfl_xor_sync(0xffffffffu, cb.m, o);
      other.found = __shfl_xor_sync(0xffffffffu, cb.found, o);
      if (mask_better(other, cb)) cb = other;
    }
    if (lane == 0) {
      s_val[wid] = cb.v;
      s_mask[wid] = cb.m;
      s_found[wid] = cb.found;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < (int)(blockDim.x / 32); ++w) {
        const MaskBest c{s_val[w], s_mask[w], s_found[w]};
        if (mask_better(c, cb)) cb = c;
      }
      // across chunks the reference keeps a chunk's best only if strictly
      // greater (a later NaN never replaces, planner.py:258-261)
      if (cb.found && (!best.found || cb.v > best.v)) best = cb;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    uint8_t* pi = out.pi + lo;
    for (int k = 0; k < L; ++k) pi[k] = best.found ? (uint8_t)((best.m >> (L - 1 - k)) & 1) : 0;
    int32_t idx[32];  // L <= 24 (planner.py:21 ORACLE_MAX_LAYERS; checked by sp_plan_exhaustive)
    finish_policy(in, inst, lo, L, idx, out, !best.found, false);
    out.status[inst] = SP_OK;
  }
}

// ---------------------------------------------------------------------------
// Eq. (1) latency (evaluator.py:64-69): one thread per instance

__global__ void eq1_kernel(sp_instances in, const double* cs, const double* ss, const double* up,
                           const double* dn, const uint8_t* pi, double* lat_out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= in.n) return;
  const int64_t lo = in.layer_off[t];
  const int64_t L = in.layer_off[t + 1] - lo;
  const double x0 = in.source_at_client[t] ? 1.0 : 0.0;
  auto term = [&](int64_t k) {
    const double x = pi[lo + k] ? 1.0 : 0.0;
    const double xp = k == 0 ? x0 : (pi[lo + k - 1] ? 1.0 : 0.0);
    // x * (c + (1 - xp) * d) + (1 - x) * (s + xp * u), numpy elementwise order
    const double a = dmul(x, dadd(cs[lo + k], dmul(dadd(1.0, -xp), dn[lo + k])));
    const double b = dmul(dadd(1.0, -x), dadd(ss[lo + k], dmul(xp, up[lo + k])));
    return dadd(a, b);
  };
  lat_out[t] = np_sum(term, L);
}

// ---------------------------------------------------------------------------
// host side

int validate(const sp_instances* in) {
  if (!in) {
    set_error(SP_ERR_INVALID, "null instance batch");
    return SP_ERR_INVALID;
  }
  if (in->n < 0 || in->total_layers < 0) {
    set_error(SP_ERR_INVALID, "negative sizes");
    return SP_ERR_INVALID;
  }
  if (in->n > 0 && (!in->layer_off || !in->client_units || !in->server_units || !in->up_units ||
                    !in->down_units || !in->r || !in->budget || !in->source_at_client)) {
    set_error(SP_ERR_INVALID, "null array in instance batch");
    return SP_ERR_INVALID;
  }
  return SP_OK;
}

int validate_out(const sp_policies* out) {
  if (!out || !out->pi || !out->client_value || !out->server_load || !out->integer_latency ||
      !out->feasible || !out->status) {
    set_error(SP_ERR_INVALID, "null array in policy batch");
    return SP_ERR_INVALID;
  }
  return SP_OK;
}

struct Carve {
  uint8_t* base;
  size_t cap, used = 0;
  void* take(size_t bytes) {
    used = align_up(used, 256);
    void* p = base + used;
    used += bytes;
    return p;
  }
};

size_t value_bytes(int mode) { return mode == VM_INT32 ? 4 : 8; }

// packed back-pointer words per stage row for rows of `cols` columns
int64_t bp_row_words_for(int mode, int64_t cols) { return ((cols + 31) / 32) * bp_words(mode); }

size_t stage_bytes_mode(int mode) {
  return align_up(kStageTile * (sizeof(StageShift) + value_bytes(mode)), 16);
}

enum DpVariant { DPV_SMEM = 0, DPV_GLOBAL = 2, DPV_STREAM = 4, DPV_STEPS = 7 };

// ---- single-CTA kernels: T x E configurations ------------------------------

constexpr int kSingleT[] = {64, 128, 256, 512, 128, 256};
constexpr int kSingleEs[] = {4, 4, 4, 4, 8, 8};  // configs 4, 5: int32 domain only
constexpr int kNumSingle = 4;

int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

// about four chunks per stage, at most 512 threads (E = 4); int32 rows up
// to 12k columns take 8 columns per thread, at most 256 threads (measured
// +3-9 % at W = 1e3-1e4, -4 % from 18k: profiles/r01/single_e8)
// (SPLITPLAN_DP_SINGLE_E = 4 or 8 forces one)
int single_cfg_for(int64_t ncol, int mode = VM_F64) {
  const int force = env_int("SPLITPLAN_DP_THREADS", 0);
  const int e = env_int("SPLITPLAN_DP_SINGLE_E", 0);
  if (mode == VM_INT32 && (e == 8 || (e == 0 && ncol <= 12288))) {
    if (force == 128) return 4;
    if (force == 256) return 5;
    return (int64_t)kSingleT[4] * 8 * 4 >= ncol ? 4 : 5;
  }
  for (int c = 0; c < kNumSingle; ++c)
    if (force == kSingleT[c]) return c;
  for (int c = 0; c < kNumSingle; ++c)
    if ((int64_t)kSingleT[c] * kSingleEs[c] * 4 >= ncol) return c;
  return kNumSingle - 1;
}
int64_t single_ch(int cfg) { return (int64_t)kSingleT[cfg] * kSingleEs[cfg]; }
int64_t single_cols(int cfg, int64_t ncol) {
  const int64_t ch = single_ch(cfg);
  return (ncol + ch - 1) / ch * ch;
}
// both rows: CH cells of NEG padding + whole chunks
size_t single_row_bytes(int mode, int64_t ncol, int cfg) {
  return 2 * (size_t)(single_ch(cfg) + single_cols(cfg, ncol)) * value_bytes(mode);
}

template <int MODE, bool SMEM, int T, int E = 4>
int launch_single_t(const DpArgs& a, int64_t n_items, size_t smem, cudaStream_t st) {
  auto kern = dp_stage_kernel<MODE, SMEM, T, E>;
  int rc = check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)kSmemCap),
                      "cudaFuncSetAttribute(dp_stage_kernel)");
  if (rc) return rc;
  kern<<<(unsigned)n_items, T, smem, st>>>(a);
  return launch_check("dp_stage_kernel launch");
}

template <int MODE, bool SMEM>
int launch_single(const DpArgs& a, int64_t n_items, int cfg, size_t smem, cudaStream_t st) {
  if (MODE == VM_INT32 && SMEM && cfg == 4) return launch_single_t<MODE, SMEM, 128, 8>(a, n_items, smem, st);
  if (MODE == VM_INT32 && SMEM && cfg == 5) return launch_single_t<MODE, SMEM, 256, 8>(a, n_items, smem, st);
  switch (cfg) {
    case 0: return launch_single_t<MODE, SMEM, 64>(a, n_items, smem, st);
    case 1: return launch_single_t<MODE, SMEM, 128>(a, n_items, smem, st);
    case 2: return launch_single_t<MODE, SMEM, 256>(a, n_items, smem, st);
    default: return launch_single_t<MODE, SMEM, 512>(a, n_items, smem, st);
  }
}

// ---- streaming (L2-resident rows, bulk-copy staged windows) ----------------

// Streaming-kernel configurations (compute threads T, columns per thread per
// chunk E, bulk-copy ring depth NSLOT), ~100 KB of ring per CTA so two CTAs
// share an SM.  The int32 domain can take 8 columns per thread (half the
// per-chunk address / barrier overhead per cell); the fp64 domains keep 4.
struct StreamCfg {
  int T, E, NSLOT;
};
constexpr StreamCfg kStreamCfgs[] = {{256, 4, 6}, {256, 8, 3}, {128, 8, 6}, {256, 4, 3}, {256, 6, 4}};
constexpr int kStreamCfgF64 = 3;
// SPLITPLAN_STREAM_CFG forces one configuration; otherwise the int32 domain
// picks between 256 x 8 and 256 x 6 per width (stream_geom), the fp64
// domains use 256 x 4.
int stream_forced_cfg(int mode) {
  if (mode != VM_INT32) return kStreamCfgF64;
  const int c = env_int("SPLITPLAN_STREAM_CFG", -1);
  return c < 0 || c > 4 || c == kStreamCfgF64 ? -1 : c;
}

int stream_threads(int cfg) { return kStreamCfgs[cfg].T; }
int64_t stream_ch(int cfg) { return (int64_t)kStreamCfgs[cfg].T * kStreamCfgs[cfg].E; }
// live rows of co-resident instances kept in L2 (SPLITPLAN_L2_BUDGET_MB).
// Measured at cfg2 (profiles/r01/stream_cfg_diag/ncu_dram_G*.csv): ~69 MB of
// rows stay resident (0.05 B/cell of DRAM reads), ~94 MB already spill
// (2.3 B/cell of DRAM reads, 6.6 B/cell of write-backs); 256 x 6 at G = 6
// (81 MB) runs fastest (profiles/r01/stream_cfg_diag/e6_k2.jsonl).
size_t l2_row_budget() {
  static size_t b = 0;
  if (!b) b = (size_t)env_int("SPLITPLAN_L2_BUDGET_MB", 90) << 20;
  return b;
}

size_t stream_smem(int mode, int cfg) {
  const size_t vb = value_bytes(mode);  // ring slots + one NEG window
  return 256 + (size_t)(kStreamCfgs[cfg].NSLOT * 4 + 1) * (stream_ch(cfg) + 16 / vb) * vb;
}
int64_t stream_span(int mode, const StreamGeom& g) {
  const int64_t line = 128 / (int64_t)value_bytes(mode);
  return (stream_ch(g.cfg) + line) + (int64_t)g.G * g.NC * stream_ch(g.cfg) + line;
}
// row buffers of the streaming kernel (profiles/r01/bufs_experiment: three
// buffers, one stage of slack, measured no faster: the L2 footprint grows by half)
constexpr int kStreamBufs = 2;
size_t stream_row_bytes(int mode, const StreamGeom& g) {
  return 2 * (size_t)kStreamBufs * (size_t)stream_span(mode, g) * value_bytes(mode);
}

template <int MODE, int T, int E, int NSLOT>
int stream_occupancy_t(int cfg) {
  auto kern = dp_stream_kernel<MODE, T, E, NSLOT, 1, 2>;
  int n = 0;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)stream_smem(MODE, cfg)) !=
          cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, T + 32, stream_smem(MODE, cfg)) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  return n > 0 ? n : 2;
}
template <int MODE>
int stream_occupancy(int cfg) {
  if (MODE != VM_INT32) return stream_occupancy_t<MODE, 256, 4, 3>(cfg);
  switch (cfg) {
    case 1: return stream_occupancy_t<MODE, 256, 8, 3>(cfg);
    case 2: return stream_occupancy_t<MODE, 128, 8, 6>(cfg);
    case 4: return stream_occupancy_t<MODE, 256, 6, 4>(cfg);
    default: return stream_occupancy_t<MODE, 256, 4, 6>(cfg);
  }
}

// co-resident streaming CTAs on this device (cached per value domain and configuration)
int stream_resident_ctas(int mode, int cfg) {
  static int cache[3][5] = {};
  if (!cache[mode][cfg]) {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
      cudaGetLastError();
      sms = 148;
    }
    const int per_sm = mode == VM_INT32 ? stream_occupancy<VM_INT32>(cfg)
                       : mode == VM_F64 ? stream_occupancy<VM_F64>(cfg)
                                        : stream_occupancy<VM_F64_NAN>(cfg);
    cache[mode][cfg] = sms * per_sm;
  }
  return cache[mode][cfg];
}

// Cluster size for one configuration: at least large enough that the rows of
// every co-resident instance fit the L2 budget; among those, the G
// minimising G * (NC * CH + sync) -- the CTA-time of one stage in columns,
// padding waste included, plus the stage-synchronisation latency per CTA
// (about 4096 columns, measured on B200).
// Returns the geometry and its cost.
StreamGeom stream_geom_cfg(int mode, int64_t ncol, int cfg, int64_t* cost) {
  const int64_t ch = stream_ch(cfg);
  const int64_t nchunks = (ncol + ch - 1) / ch;
  const int resident = stream_resident_ctas(mode, cfg);
  const int force = env_int("SPLITPLAN_DP_CLUSTER", 0);
  auto geom = [&](int G) {
    StreamGeom t{G, (int)((nchunks + G - 1) / G), 0, 0, 0, cfg};
    t.G = (int)((nchunks + t.NC - 1) / t.NC);
    return t;
  };
  const int64_t sync = 4096;
  auto cost_of = [&](const StreamGeom& t) { return (int64_t)t.G * ((int64_t)t.NC * ch + sync); };
  if (force >= 1 && force <= 16) {
    const StreamGeom t = geom(force);
    *cost = cost_of(t);
    return t;
  }
  int gmin = 16;
  for (int G = 1; G <= 16; ++G)
    if ((size_t)(resident / G) * stream_row_bytes(mode, geom(G)) <= l2_row_budget()) {
      gmin = G;
      break;
    }
  StreamGeom best = geom(gmin);
  for (int G = gmin + 1; G <= 16; ++G) {
    const StreamGeom t = geom(G);
    if (cost_of(t) < cost_of(best)) best = t;
  }
  *cost = cost_of(best);
  return best;
}
StreamGeom stream_geom(int mode, int64_t ncol) {
  const int forced = stream_forced_cfg(mode);
  int64_t c1 = 0, c2 = 0;
  if (forced >= 0) return stream_geom_cfg(mode, ncol, forced, &c1);
  const StreamGeom e8 = stream_geom_cfg(mode, ncol, 1, &c1);
  const StreamGeom e6 = stream_geom_cfg(mode, ncol, 4, &c2);
  return c2 < c1 ? e6 : e8;
}

template <int MODE, int T, int E, int NSLOT, int NI, int NBUF>
int launch_stream_t(const DpArgs& a, int64_t n_items, StreamGeom geo, cudaStream_t st) {
  auto kern = dp_stream_kernel<MODE, T, E, NSLOT, NI, NBUF>;
  const size_t smem = stream_smem(MODE, geo.cfg);
  int rc = check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                      "cudaFuncSetAttribute(dp_stream_kernel)");
  if (rc) return rc;
  if (geo.G > 8) {
    rc = check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
                    "cudaFuncSetAttribute(non-portable cluster)");
    if (rc) return rc;
  }
  geo.n_items = (int)n_items;
  geo.row_hint = env_int("SPLITPLAN_ROW_EVICT_LAST", 0) ? 1 : 0;
  geo.diag = env_int("SPLITPLAN_STREAM_DIAG", 0);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((n_items + NI - 1) / NI * geo.G), 1, 1);
  cfg.blockDim = dim3((unsigned)(T + 32), 1, 1);  // + the producer warp
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)geo.G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  rc = check_cuda(cudaLaunchKernelEx(&cfg, kern, a, geo), "dp_stream_kernel launch");
  if (rc) return rc;
  return launch_check("dp_stream_kernel launch");
}
template <int MODE>
int launch_stream(const DpArgs& a, int64_t n_items, StreamGeom geo, cudaStream_t st) {
  if (MODE == VM_INT32 && geo.cfg == 1) return launch_stream_t<MODE, 256, 8, 3, 1, 2>(a, n_items, geo, st);
  if (MODE == VM_INT32 && geo.cfg == 4) return launch_stream_t<MODE, 256, 6, 4, 1, 2>(a, n_items, geo, st);
  if (MODE == VM_INT32 && geo.cfg == 2) return launch_stream_t<MODE, 128, 8, 6, 1, 2>(a, n_items, geo, st);
  constexpr int NS = MODE == VM_INT32 ? 6 : 3;
  return launch_stream_t<MODE, 256, 4, NS, 1, kStreamBufs>(a, n_items, geo, st);
}

// SPLITPLAN_TRACE=1: host-side phase timestamps of run_dp on stderr
struct Trace {
  bool on = env_int("SPLITPLAN_TRACE", 0) != 0;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void operator()(const char* what, long long x = -1) const {
    if (!on) return;
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    fprintf(stderr, "[splitplan trace] %9.3f ms  %s %lld\n", ms, what, x);
  }
};

// ---- breakpoint-list kernels ------------------------------------------------

// tier geometry: warps (instances) per block
#ifndef SP_STEPS_WPB
#define SP_STEPS_WPB 3
#endif
template <int CAP> constexpr int steps_wpb() { return CAP >= 1024 ? 1 : SP_STEPS_WPB; }
size_t steps_smem(int mode, int cap) {
  const int WPB = cap >= 1024 ? 1 : SP_STEPS_WPB;
  return (size_t)WPB * steps_arrays_rt(cap) * (size_t)cap *
         (mode == VM_INT32 ? sizeof(Ent<VM_INT32>) : sizeof(Ent<VM_F64>));
}

template <int MODE, int CAP>
int launch_steps_t(const StepsArgs& sa, cudaStream_t st) {
  constexpr int WPB = steps_wpb<CAP>();
  auto kern = dp_steps_kernel<MODE, CAP, WPB>;
  const size_t smem = steps_smem(MODE, CAP);
  int rc = check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                      "cudaFuncSetAttribute(dp_steps_kernel)");
  if (rc) return rc;
  kern<<<(unsigned)((sa.n_items + WPB - 1) / WPB), WPB * 32, smem, st>>>(sa);
  return launch_check("dp_steps_kernel launch");
}
// K2 + K3 on breakpoint lists; `out` null: forward pass only
int launch_steps(int mode, int cap, StepsArgs sa, const sp_instances* in, const sp_policies* out, int32_t* idx,
                 cudaStream_t st) {
  if (sa.n_items == 0) return SP_OK;
  sa.walk = out ? 1 : 0;
  if (in) sa.in = *in;
  if (out) sa.out = *out;
  sa.idx = idx;
  if (cap == kStepsCap)
    return mode == VM_INT32 ? launch_steps_t<VM_INT32, kStepsCap>(sa, st) : launch_steps_t<VM_F64, kStepsCap>(sa, st);
  return mode == VM_INT32 ? launch_steps_t<VM_INT32, kStepsCapWide>(sa, st)
                          : launch_steps_t<VM_F64, kStepsCapWide>(sa, st);
}

int forced_variant() {
  const char* v = getenv("SPLITPLAN_DP_VARIANT");
  if (!v) return -1;
  if (!strcmp(v, "smem")) return DPV_SMEM;
  if (!strcmp(v, "global")) return DPV_GLOBAL;
  if (!strcmp(v, "stream")) return DPV_STREAM;
  if (!strcmp(v, "grid")) return 5;  // DPV_GRID
  if (!strcmp(v, "steps")) return DPV_STEPS;
  return -1;
}

// Launch plan of one instance: kernel variant, its configuration, and the
// workspace / shared memory it needs.
struct DpPlan {
  int variant = DPV_SMEM;
  int cfg = 0;                  // single-CTA T x E configuration; breakpoint-list capacity (DPV_STEPS)
  int threads = 0;
  StreamGeom sgeo{0, 0, 0, 0};  // stream
  size_t bp = 0, rows = 0, smem = 0;
  int64_t bp_row_words = 0;
  // launches sharing a key go out together
  bool same_launch(const DpPlan& o) const {
    return variant == o.variant && cfg == o.cfg && threads == o.threads && sgeo.G == o.sgeo.G &&
           sgeo.NC == o.sgeo.NC && sgeo.cfg == o.sgeo.cfg;
  }
};

// The widest row the single-CTA kernel holds in shared memory (it runs at
// ~1e12 cells/s there, profiles/r01/single_e8): narrower rows stay on it.
int64_t smem_max_cols(int mode) {
  auto fits = [&](int64_t ncol) {
    return single_row_bytes(mode, ncol, single_cfg_for(ncol, mode)) + stage_bytes_mode(mode) <= kSmemCap;
  };
  int64_t lo = 1, hi = (int64_t)1 << 20;  // fits(lo), !fits(hi)
  while (hi - lo > 1) {
    const int64_t m = (lo + hi) / 2;
    if (fits(m)) lo = m;
    else hi = m;
  }
  return lo;
}
// narrowest row the breakpoint lists take (all of them when forced)
// (rows of any width: on model-derived instances the lists beat the SMEM
// kernel down to the narrowest rows -- cfg4 solve 349 ms at a 1,024-column
// threshold, 221 ms at 32, profiles/r02/tier0/threshold.md -- and a row of at
// most CAP columns cannot overflow them; SPLITPLAN_STEPS_MIN_COLS moves it)
constexpr int64_t kStepsMinCols = 0;
int64_t steps_min_cols(int mode, int force) {
  (void)mode;
  if (force == DPV_STEPS) return 0;
  const int v = env_int("SPLITPLAN_STEPS_MIN_COLS", -1);
  return v >= 0 ? v : kStepsMinCols;
}

// steps_eligible: the breakpoint-list kernels may take the instance: rows
// wider than one SM's shared memory (where the dense alternative is the
// L2-streaming kernel) and narrower than the whole-GPU path, not for full
// tables, not in the NaN domain
// (lo_i32 / lo_f64: steps_min_cols of the two domains, computed once per call)
bool steps_eligible(int mode, int64_t ncol, int force, bool tables, int64_t lo_i32, int64_t lo_f64) {
  return !tables && mode != VM_F64_NAN && ncol < kGridMinColsSteps &&
         ncol >= (mode == VM_INT32 ? lo_i32 : lo_f64) && (force < 0 || force == DPV_STEPS);
}

// `steps_cap` > 0: plan the breakpoint-list kernel with that capacity (the
// caller checked steps_eligible); 0: a dense kernel.
DpPlan plan_instance(int mode, int64_t L, int64_t ncol, int force, bool tables, int steps_cap = 0) {
  DpPlan p;
  if (steps_cap > 0) {
    p.variant = DPV_STEPS;
    p.cfg = steps_cap;
    p.threads = (steps_cap >= 1024 ? 1 : SP_STEPS_WPB) * 32;
    p.smem = steps_smem(mode, steps_cap);
    p.bp = align_up(steps_store_bytes((int)L, steps_cap), 256);
    return p;
  }
  const size_t vb = value_bytes(mode);
  p.cfg = single_cfg_for(ncol, (force == DPV_GLOBAL || tables) ? VM_F64 : mode);
  const size_t single_rows = single_row_bytes(mode, ncol, p.cfg);
  const bool fits_cta = single_rows + stage_bytes_mode(mode) <= kSmemCap;
  if (force == DPV_GLOBAL || (tables && force < 0)) p.variant = DPV_GLOBAL;
  else if (force == DPV_SMEM && fits_cta) p.variant = DPV_SMEM;
  else if (force == DPV_STREAM) p.variant = DPV_STREAM;
  else if (fits_cta) p.variant = DPV_SMEM;
  else p.variant = DPV_STREAM;

  switch (p.variant) {
    case DPV_SMEM:
    case DPV_GLOBAL:
      p.threads = kSingleT[p.cfg];
      p.bp_row_words = bp_row_words_for(mode, single_cols(p.cfg, ncol));
      p.rows = p.variant == DPV_GLOBAL ? align_up(single_rows, 256) : 0;
      p.smem = stage_bytes_mode(mode) + (p.variant == DPV_SMEM ? single_rows : 0);
      break;
    case DPV_STREAM:
      p.sgeo = stream_geom(mode, ncol);
      p.threads = stream_threads(p.sgeo.cfg);
      p.bp_row_words = bp_row_words_for(mode, (int64_t)p.sgeo.G * p.sgeo.NC * stream_ch(p.sgeo.cfg));
      p.rows = align_up(stream_row_bytes(mode, p.sgeo), 256);
      p.smem = stream_smem(mode, p.sgeo.cfg);
      break;
  }
  p.bp = align_up((size_t)L * (size_t)p.bp_row_words * 4, 256);
  return p;
}

// ---- tier 0: the SMEM kernel's instances, planned on the device -------------
//
// Rows narrow enough for one CTA's shared memory run on dp_stage_kernel<SMEM>
// (~1e12 cells/s).  A batch of millions of them (configs[3]: 4.2M requests)
// used to be planned instance by instance on the host; tier 0 plans them on
// the device instead: t0_count_kernel classifies every instance by launch
// configuration (value domain x T x E, the default rule of single_cfg_for)
// and counts instances, cells and back-pointer bytes per class; after the one
// synchronisation the call makes anyway, t0_scatter_kernel writes each
// instance's work item into its class's segment of the work list and carves
// its back-pointer table out of the workspace with a warp-aggregated bump
// allocator; then one dp_stage_kernel and one backtrack_kernel per non-empty
// class.  Placement order is irrelevant to the results (each instance's table
// is its own).
constexpr int kT0Classes = 11;  // int32: cfg 4, 5, 3; fp64 and NaN domain: cfg 0-3
constexpr int kT0Block = 256;   // instances per counting block (the unit waves are cut at)
struct T0Stats {                // global: [max_ncol | class cursors | bump]
  unsigned long long max_ncol[kT0Classes];
  unsigned long long cursor[kT0Classes];
  unsigned long long bump;
};
struct T0Block {  // per counting block
  uint32_t count[kT0Classes];
  uint32_t pad;
  unsigned long long bytes;  // back-pointer bytes (each table 256-B aligned)
  unsigned long long cells[kT0Classes];
};
struct T0Seg {  // a wave's class segments in the work list
  unsigned long long off[kT0Classes];
};
__host__ __device__ inline int t0_class_mode(int c) { return c < 3 ? VM_INT32 : (c < 7 ? VM_F64 : VM_F64_NAN); }
__host__ __device__ inline int t0_class_cfg(int c) {
  return c < 3 ? (c == 0 ? 4 : (c == 1 ? 5 : 3)) : (c < 7 ? c - 3 : c - 7);
}
// single_cfg_for without the environment overrides (tier 0 is off when one is set)
__host__ __device__ inline int t0_cfg_of(int64_t ncol, int mode) {
  if (mode == VM_INT32 && ncol <= 12288) return 128 * 8 * 4 >= ncol ? 4 : 5;
  if (ncol <= 64 * 4 * 4) return 0;
  if (ncol <= 128 * 4 * 4) return 1;
  if (ncol <= 256 * 4 * 4) return 2;
  return 3;
}
__host__ __device__ inline int t0_class_of(int64_t ncol, int mode) {
  const int cfg = t0_cfg_of(ncol, mode);
  if (mode == VM_INT32) return cfg == 4 ? 0 : (cfg == 5 ? 1 : 2);
  return (mode == VM_F64 ? 3 : 7) + cfg;
}
__host__ __device__ inline int64_t t0_ch(int cfg) {
  constexpr int T[] = {64, 128, 256, 512, 128, 256}, E[] = {4, 4, 4, 4, 8, 8};
  return (int64_t)T[cfg] * E[cfg];
}
__host__ __device__ inline int64_t t0_row_words(int mode, int cfg, int64_t ncol) {
  const int64_t ch = t0_ch(cfg), cols = (ncol + ch - 1) / ch * ch;
  return (cols + 31) / 32 * bp_words(mode);
}
// class and back-pointer bytes of instance k (class -1: not tier 0)
// (skip: the query's stand-in for tier 1's flags -- rows in [skip[mode], skip[2])
// outside the NaN domain are tier 1's)
__device__ __forceinline__ int t0_classify(const sp_instances& in, const InstInfo* info, const int32_t* flag,
                                           int64_t max_i32, int64_t max_f64, const int64_t* skip, int64_t k,
                                           int64_t& ncol, unsigned long long& bytes, unsigned long long& cells) {
  const InstInfo inf = info[k];
  ncol = inf.w_eff + 1;
  const int64_t L = in.layer_off[k + 1] - in.layer_off[k];
  bytes = cells = 0;
  if ((flag && !flag[k]) || L <= 0 || ncol > (inf.mode == VM_INT32 ? max_i32 : max_f64)) return -1;
  if (inf.mode != VM_F64_NAN && ncol < skip[2] && ncol >= skip[inf.mode == VM_INT32 ? 0 : 1]) return -1;
  const int c = t0_class_of(ncol, inf.mode);
  bytes = align_up((size_t)L * (size_t)t0_row_words(inf.mode, t0_class_cfg(c), ncol) * 4, 256);
  cells = (unsigned long long)L * (unsigned long long)ncol;
  return c;
}

// one thread per instance: per-block class counts, cells and back-pointer
// bytes (the host cuts waves at block boundaries), global widest row per class
struct T0Skip {
  int64_t v[3];  // [lo int32, lo fp64, hi]; hi = 0: nothing skipped
};
__global__ void __launch_bounds__(kT0Block) t0_count_kernel(sp_instances in, const InstInfo* info,
                                                            const int32_t* flag, int64_t max_i32, int64_t max_f64,
                                                            T0Skip skip, uint8_t* cls, T0Stats* stats,
                                                            T0Block* blocks) {
  __shared__ uint32_t s_cnt[kT0Classes];
  __shared__ unsigned long long s_cells[kT0Classes], s_max[kT0Classes], s_bytes;
  if (threadIdx.x < kT0Classes) {
    s_cnt[threadIdx.x] = 0;
    s_cells[threadIdx.x] = 0;
    s_max[threadIdx.x] = 0;
  }
  if (threadIdx.x == 0) s_bytes = 0;
  __syncthreads();
  const int64_t k = (int64_t)blockIdx.x * kT0Block + threadIdx.x;
  if (k < in.n) {
    int64_t ncol;
    unsigned long long bytes, cells;
    const int c = t0_classify(in, info, flag, max_i32, max_f64, skip.v, k, ncol, bytes, cells);
    cls[k] = c < 0 ? 255 : (uint8_t)c;
    if (c >= 0) {
      atomicAdd(&s_cnt[c], 1u);
      atomicAdd(&s_cells[c], cells);
      atomicMax(&s_max[c], (unsigned long long)ncol);
      atomicAdd(&s_bytes, bytes);
    }
  }
  __syncthreads();
  T0Block& b = blocks[blockIdx.x];
  if (threadIdx.x < kT0Classes) {
    b.count[threadIdx.x] = s_cnt[threadIdx.x];
    b.cells[threadIdx.x] = s_cells[threadIdx.x];
    if (s_max[threadIdx.x]) atomicMax(&stats->max_ncol[threadIdx.x], s_max[threadIdx.x]);
  }
  if (threadIdx.x == 0) {
    b.pad = 0;
    b.bytes = s_bytes;
  }
}

// one wave (counting blocks [b0, b0 + gridDim.x)): the work items into their
// class segments, back-pointer tables carved from `bump` (warp-aggregated),
// the instances' flags cleared (solved here)
__global__ void __launch_bounds__(kT0Block) t0_scatter_kernel(sp_instances in, const InstInfo* info,
                                                              const uint8_t* cls, int64_t b0, T0Seg seg,
                                                              T0Stats* stats, DpWork* work, int32_t* flag) {
  const int lane = threadIdx.x & 31;
  const int64_t k = (b0 + blockIdx.x) * kT0Block + threadIdx.x;
  const int c = k < in.n && cls[k] != 255 ? (int)cls[k] : -1;
  unsigned long long bytes = 0;
  int64_t ncol = 0;
  int mode = 0;
  if (c >= 0) {
    const InstInfo inf = info[k];
    ncol = inf.w_eff + 1;
    mode = inf.mode;
    const int64_t L = in.layer_off[k + 1] - in.layer_off[k];
    bytes = align_up((size_t)L * (size_t)t0_row_words(mode, t0_class_cfg(c), ncol) * 4, 256);
  }
  unsigned long long incl = bytes;  // exclusive scan of the warp's bytes + one bump
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  unsigned long long wbase = 0;
  if (lane == 31 && incl) wbase = atomicAdd(&stats->bump, incl);
  wbase = __shfl_sync(0xffffffffu, wbase, 31);
  const unsigned peers = __match_any_sync(0xffffffffu, c);  // one cursor increment per class in the warp
  const int leader = __ffs(peers) - 1;
  unsigned long long pbase = 0;
  if (c >= 0 && lane == leader) pbase = atomicAdd(&stats->cursor[c], (unsigned long long)__popc(peers));
  pbase = __shfl_sync(peers, pbase, leader);
  if (c >= 0) {
    DpWork w;
    w.inst = k;
    w.bp_off = (int64_t)(wbase + incl - bytes);
    w.row_off = -1;
    w.bp_row_words = t0_row_words(mode, t0_class_cfg(c), ncol);
    work[seg.off[c] + pbase + __popc(peers & ((1u << lane) - 1u))] = w;
    if (flag) flag[k] = 0;
  }
}

int launch_plan(int mode, const DpPlan& p, const DpArgs& a, int64_t n_items, cudaStream_t st,
                const sp_instances* in = nullptr, const sp_policies* out = nullptr, int32_t* idx = nullptr) {
  if (n_items == 0) return SP_OK;
  switch (p.variant) {
    case DPV_STEPS: {
      StepsArgs sa = {};
      sa.layer_off = a.layer_off;
      sa.sac = a.sac;
      sa.info = a.info;
      sa.shifts = a.shifts;
      sa.rv = a.rv;
      sa.work = a.work;
      sa.store = a.bp;
      sa.overflow = a.overflow;
      sa.n_items = n_items;
      return launch_steps(mode, p.cfg, sa, in, out, idx, st);
    }
    case DPV_STREAM:
      switch (mode) {
        case VM_INT32: return launch_stream<VM_INT32>(a, n_items, p.sgeo, st);
        case VM_F64: return launch_stream<VM_F64>(a, n_items, p.sgeo, st);
        default: return launch_stream<VM_F64_NAN>(a, n_items, p.sgeo, st);
      }
    default: {
      const bool sm = p.variant == DPV_SMEM;
      switch (mode * 2 + (sm ? 1 : 0)) {
        case VM_INT32 * 2 + 1: return launch_single<VM_INT32, true>(a, n_items, p.cfg, p.smem, st);
        case VM_INT32 * 2 + 0: return launch_single<VM_INT32, false>(a, n_items, p.cfg, p.smem, st);
        case VM_F64 * 2 + 1: return launch_single<VM_F64, true>(a, n_items, p.cfg, p.smem, st);
        case VM_F64 * 2 + 0: return launch_single<VM_F64, false>(a, n_items, p.cfg, p.smem, st);
        case VM_F64_NAN * 2 + 1: return launch_single<VM_F64_NAN, true>(a, n_items, p.cfg, p.smem, st);
        default: return launch_single<VM_F64_NAN, false>(a, n_items, p.cfg, p.smem, st);
      }
    }
  }
}

// algorithmic HBM bytes per DP cell of a variant: rows on chip or in L2 ->
// the packed back-pointer bits only; global rows of the single-CTA kernel ->
// read + write of both rows plus those bits
double hbm_bytes_per_cell(int mode, int variant) {
  const double bits = bp_words(mode) * 4.0 / 32.0;
  if (variant == DPV_STEPS) return 0.0;  // list bytes depend on the data, not the cells
  return variant == DPV_GLOBAL ? 4.0 * (double)value_bytes(mode) + bits : bits;
}

// ---- grid path: one huge instance over the whole GPU --------------------------

// grid kernel configuration: 256 threads; int32 rows 6 columns per thread and
// a 4-slot ring (the streaming kernel's cfg2 geometry), fp64 4 and 3 slots
constexpr int kGridT = 256;
template <int MODE> constexpr int grid_e() { return MODE == VM_INT32 ? 6 : 4; }
template <int MODE> constexpr int grid_slots() { return MODE == VM_INT32 ? 4 : 3; }
inline int grid_e_rt(int mode) { return mode == VM_INT32 ? 6 : 4; }
inline int grid_slots_rt(int mode) { return mode == VM_INT32 ? 4 : 3; }
inline int64_t grid_ch(int mode) { return (int64_t)kGridT * grid_e_rt(mode); }
constexpr int64_t kGridMinCols = (int64_t)1 << 22;
enum { DPV_GRID = 5 };

size_t grid_smem(int mode) {
  const size_t vb = value_bytes(mode);  // ring slots + one NEG window
  return 256 + (size_t)(grid_slots_rt(mode) * 4 + 1) * (grid_ch(mode) + 16 / vb) * vb;
}

template <int MODE>
int grid_resident() {
  auto kern = dp_grid_kernel<MODE, kGridT, grid_e<MODE>(), grid_slots<MODE>()>;
  int n = 0, dev = 0, sms = 148;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)grid_smem(MODE)) !=
          cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, kGridT + 32, grid_smem(MODE)) != cudaSuccess ||
      cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n * sms;
}

template <int MODE>
int launch_grid_t(const GridArgs& g, cudaStream_t st) {
  auto kern = dp_grid_kernel<MODE, kGridT, grid_e<MODE>(), grid_slots<MODE>()>;
  // per device: a partition may be launched on a peer device
  int rc0 = check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)grid_smem(MODE)),
                       "cudaFuncSetAttribute(dp_grid_kernel)");
  if (rc0) return rc0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(g.G * g.launch_parts), 1, 1);  // every partition of this launch
  cfg.blockDim = dim3((unsigned)(kGridT + 32), 1, 1);
  cfg.dynamicSmemBytes = grid_smem(MODE);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // every CTA co-resident: the waits are safe
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int rc = check_cuda(cudaLaunchKernelEx(&cfg, kern, g), "dp_grid_kernel launch");
  if (rc) return rc;
  return launch_check("dp_grid_kernel launch");
}

int launch_grid(int mode, const GridArgs& g, cudaStream_t st) {
  switch (mode) {
    case VM_INT32: return launch_grid_t<VM_INT32>(g, st);
    case VM_F64: return launch_grid_t<VM_F64>(g, st);
    default: return launch_grid_t<VM_F64_NAN>(g, st);
  }
}

// ---- capacity partitions: geometry, partition workspaces, phases -----------

// Geometry of one huge instance split into `nparts` capacity partitions of G
// CTAs each, and the layout of ONE partition's workspace (the same for every
// partition; each partition's lives on that partition's device):
//   [stage records: shifts L x 16 B | values L x 8 B | frontiers L x 8 B]
//   [progress counters G x 4 B][state 128 B][rows 3 x (C, S) x span]
//   [checkpoint rows nckpt x (C, S) x Wp][back-pointers K stages x row_words]
// Checkpoint c holds row seg_begin(c) of the partition's own columns
// (c = 1..nseg; nseg = 1 keeps only the final row).
struct GridGeom {
  int mode = 0, L = 0, G = 1, NC = 1, nparts = 1, K = 1, nseg = 1, nckpt = 2, sac = 0;
  int64_t ncol = 0, B = 0, Wp = 0, halo = 0, span = 0, row_words = 0;
  size_t rec_off = 0, prog_off = 0, state_off = 0, rows_off = 0, ckpt_off = 0, bp_off = 0;
  size_t ckpt_bytes = 0, bp_stage = 0, part_bytes = 0;
  int seg_begin(int sg) const { return sg == 0 ? 0 : L - (nseg - sg) * K; }  // seg_begin(nseg) == L
  int owner_part() const { return (int)((ncol - 1) / Wp); }                 // partition of column W_eff
  // pointers into one partition workspace
  StageShift* shifts(uint8_t* pw) const { return (StageShift*)(pw + rec_off); }
  int64_t* rv(uint8_t* pw) const { return (int64_t*)(pw + rec_off + (size_t)L * sizeof(StageShift)); }
  int2* reach(uint8_t* pw) const {
    return (int2*)(pw + rec_off + (size_t)L * (sizeof(StageShift) + sizeof(int64_t)));
  }
  uint32_t* prog(uint8_t* pw) const { return (uint32_t*)(pw + prog_off); }
  int64_t* state(uint8_t* pw) const { return (int64_t*)(pw + state_off); }
  InstInfo* info(uint8_t* pw) const { return (InstInfo*)(pw + state_off + 64); }
  uint8_t* ckpt(uint8_t* pw, int c) const { return pw + ckpt_off + (size_t)c * ckpt_bytes; }
  uint32_t* bp(uint8_t* pw) const { return (uint32_t*)(pw + bp_off); }
};

void grid_layout(GridGeom& g, int K) {
  const size_t vb = value_bytes(g.mode);
  g.K = K;
  g.nseg = (g.L + K - 1) / K;
  g.nckpt = g.nseg + 1;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o = align_up(o + bytes, 256);
    return at;
  };
  g.rec_off = take((size_t)g.L * (sizeof(StageShift) + sizeof(int64_t) + sizeof(int2)));
  g.prog_off = take((size_t)g.G * 4);
  g.state_off = take(128);
  g.rows_off = take(2 * (size_t)kRowBufs * (size_t)g.span * vb);
  g.ckpt_bytes = align_up(2 * (size_t)g.Wp * vb, 256);
  g.ckpt_off = take((size_t)g.nckpt * g.ckpt_bytes);
  g.bp_stage = (size_t)g.row_words * 4;
  g.bp_off = take((size_t)K * g.bp_stage);
  g.part_bytes = o;
}

int grid_resident_rt(int mode) {
  return mode == VM_INT32 ? grid_resident<VM_INT32>()
         : mode == VM_F64 ? grid_resident<VM_F64>()
                          : grid_resident<VM_F64_NAN>();
}

// Capacity partitions and segment length for one instance: `ctas` CTAs per
// partition at most (what stays co-resident on its device), every partition
// workspace at most `avail` bytes.  Sets *too_wide when a stage's read-back
// spans a whole partition (the halo would be the partition): use one.
// SP_ERR_WORKSPACE (with the required bytes) when even checkpointing at the
// smallest footprint does not fit.
int grid_geometry(int mode, int L, int64_t ncol, int nparts, int ctas, int max_shift, size_t avail,
                  int force_k, GridGeom* out, bool* too_wide) {
  GridGeom g;
  g.mode = mode;
  g.L = L;
  g.ncol = ncol;
  *too_wide = false;
  const int64_t ch = grid_ch(mode), line = 128 / (int64_t)value_bytes(mode);
  const int64_t nchunks = (ncol + ch - 1) / ch;
  nparts = (int)std::max<int64_t>(1, std::min<int64_t>(std::min(nparts, kMaxParts), nchunks));
  int G = (int)std::max<int64_t>(1, std::min<int64_t>(std::max(ctas, 1), (nchunks + nparts - 1) / nparts));
  const int NC = (int)((nchunks + (int64_t)G * nparts - 1) / ((int64_t)G * nparts));
  G = (int)((nchunks + (int64_t)NC * nparts - 1) / ((int64_t)NC * nparts));
  nparts = (int)((nchunks + (int64_t)NC * G - 1) / ((int64_t)NC * G));  // no partition left empty
  g.G = G;
  g.NC = NC;
  g.nparts = nparts;
  g.B = (int64_t)NC * ch;
  g.Wp = (int64_t)G * g.B;
  if (nparts > 1) {  // the widest read-back of any stage plus alignment slack, whole lines
    g.halo = ((int64_t)max_shift + 2 * line + line - 1) / line * line;
    if (g.halo > g.Wp) {
      *too_wide = true;
      return SP_OK;
    }
  }
  g.span = (ch + line) + g.halo + g.Wp + line;
  g.row_words = bp_row_words_for(mode, g.Wp);
  auto need = [&](int k) {
    GridGeom t = g;
    grid_layout(t, k);
    return t.part_bytes;
  };
  int K = force_k > 0 ? std::min(force_k, L) : L;
  if (force_k <= 0 && need(K) > avail) {
    // footprint ~ nseg checkpoints + K back-pointer stages: smallest near
    // K = sqrt(L * ckpt / bp); above that it grows with K.  Take the longest
    // segments that fit.
    GridGeom t = g;
    grid_layout(t, 1);
    int kopt = (int)std::max(1.0, std::sqrt((double)L * (double)t.ckpt_bytes / (double)t.bp_stage));
    kopt = std::min(kopt, L);
    K = kopt;
    if (need(kopt) <= avail) {
      int lo = kopt, hi = L;  // need(lo) fits, need(hi) does not
      while (hi - lo > 1) {
        const int mid = lo + (hi - lo) / 2;
        if (need(mid) <= avail) lo = mid;
        else hi = mid;
      }
      K = lo;
    }
  }
  grid_layout(g, K);
  *out = g;
  if (g.part_bytes > avail) {
    set_required_workspace(g.part_bytes);
    set_error(SP_ERR_WORKSPACE, "capacity partition (%d stages x %lld columns) needs %zu B of workspace, %zu B available",
              L, (long long)g.Wp, g.part_bytes, avail);
    return SP_ERR_WORKSPACE;
  }
  return SP_OK;
}

// Launch arguments of one phase: stages [k0, k0 + cnt) from checkpoint
// `init_ckpt` (0: the origin row), writing checkpoint `out_ckpt` (0: none),
// keeping the back-pointers when `keep_bp`.  pw[p]: partition p's workspace
// as seen from the launching device (peers through peer access / IPC).
GridArgs grid_args(const GridGeom& g, uint8_t* const* pw, int k0, int cnt, int init_ckpt, int out_ckpt,
                   bool keep_bp, int sys) {
  GridArgs a = {};
  a.k_begin = k0;
  a.k_count = cnt;
  a.ncol = (int)g.ncol;
  a.G = g.G;
  a.NC = g.NC;
  a.sac = g.sac;
  a.bp_row_words = g.row_words;
  a.nparts = g.nparts;
  a.part_base = 0;
  a.launch_parts = g.nparts;
  a.sys = sys;
  a.halo = (int)g.halo;
  for (int p = 0; p < g.nparts; ++p) {
    GridPart& q = a.parts[p];
    if (!pw[p]) continue;  // not mapped in this process: never touched by this launch
    q.rows = pw[p] + g.rows_off;
    q.prog = g.prog(pw[p]);
    q.bp = keep_bp ? g.bp(pw[p]) : nullptr;
    q.init = init_ckpt > 0 ? g.ckpt(pw[p], init_ckpt) : nullptr;
    q.init_left = (init_ckpt > 0 && p > 0 && pw[p - 1]) ? g.ckpt(pw[p - 1], init_ckpt) : nullptr;
    q.out = out_ckpt > 0 ? g.ckpt(pw[p], out_ckpt) : nullptr;
  }
  return a;
}

// the stage records a launch on partition p's device reads (its own copy)
void grid_set_records(GridArgs& a, const GridGeom& g, uint8_t* pw, bool use_reach) {
  a.shifts = g.shifts(pw);
  a.rv = g.rv(pw);
  a.reach = use_reach ? g.reach(pw) : nullptr;
}

// One instance solved over capacity partitions inside this process (one
// device, or one device per partition).  Owns the per-partition streams and
// events; every partition workspace is the caller's.
struct GridRun {
  GridGeom g;
  int cur = 0;
  int dev[kMaxParts] = {};
  uint8_t* pw[kMaxParts] = {};
  bool separate = false, multi = false, use_reach = true;
  int sys = 0;
  cudaStream_t pst[kMaxParts] = {};
  cudaEvent_t ev[kMaxParts] = {};
  cudaEvent_t zev[kMaxParts] = {};
  cudaEvent_t start = nullptr;
  ~GridRun() {
    for (int p = 0; p < kMaxParts; ++p) {
      if (!pst[p]) continue;
      cudaSetDevice(dev[p]);
      cudaStreamSynchronize(pst[p]);
      cudaStreamDestroy(pst[p]);
      if (ev[p]) cudaEventDestroy(ev[p]);
      if (zev[p]) cudaEventDestroy(zev[p]);
    }
    cudaSetDevice(cur);
    if (start) cudaEventDestroy(start);
  }
  int init_streams() {
    int rc = check_cuda(cudaEventCreateWithFlags(&start, cudaEventDisableTiming), "event");
    for (int p = 0; p < g.nparts && !rc; ++p) {
      cudaSetDevice(dev[p]);
      rc = check_cuda(cudaStreamCreateWithFlags(&pst[p], cudaStreamNonBlocking), "partition stream");
      if (!rc) rc = check_cuda(cudaEventCreateWithFlags(&ev[p], cudaEventDisableTiming), "event");
      if (!rc) rc = check_cuda(cudaEventCreateWithFlags(&zev[p], cudaEventDisableTiming), "event");
    }
    cudaSetDevice(cur);
    return rc;
  }
  // forward / recompute phase over every partition, stream-ordered after st
  int phase(int k0, int cnt, int init_ckpt, int out_ckpt, bool keep_bp, cudaStream_t st) {
    GridArgs a = grid_args(g, pw, k0, cnt, init_ckpt, out_ckpt, keep_bp, sys);
    int rc;
    if (!separate) {  // one launch covers every partition (all on this device)
      for (int p = 0; p < g.nparts; ++p) {
        rc = check_cuda(cudaMemsetAsync(g.prog(pw[p]), 0, (size_t)g.G * 4, st), "zero progress counters");
        if (rc) return rc;
      }
      grid_set_records(a, g, pw[0], use_reach);
      return launch_grid(g.mode, a, st);
    }
    // one launch per partition, all in flight together; every partition's
    // counters are zero before any partition starts
    rc = check_cuda(cudaEventRecord(start, st), "record phase start");
    for (int p = 0; p < g.nparts && !rc; ++p) {
      cudaSetDevice(dev[p]);
      rc = check_cuda(cudaStreamWaitEvent(pst[p], start, 0), "partition wait");
      if (!rc) rc = check_cuda(cudaMemsetAsync(g.prog(pw[p]), 0, (size_t)g.G * 4, pst[p]), "zero counters");
      if (!rc) rc = check_cuda(cudaEventRecord(zev[p], pst[p]), "record counters zeroed");
    }
    for (int p = 0; p < g.nparts && !rc; ++p) {
      cudaSetDevice(dev[p]);
      for (int q = 0; q < g.nparts && !rc; ++q) rc = check_cuda(cudaStreamWaitEvent(pst[p], zev[q], 0), "wait");
      GridArgs ap = a;
      ap.part_base = p;
      ap.launch_parts = 1;
      grid_set_records(ap, g, pw[p], use_reach);
      if (!rc) rc = launch_grid(g.mode, ap, pst[p]);
      if (!rc) rc = check_cuda(cudaEventRecord(ev[p], pst[p]), "record partition end");
    }
    cudaSetDevice(cur);
    for (int p = 0; p < g.nparts && !rc; ++p) rc = check_cuda(cudaStreamWaitEvent(st, ev[p], 0), "join partitions");
    return rc;
  }
  // backtrack through segment sg, partitions right to left, each on its own
  // device reading its own back-pointers; (j, side, next stage) handed over
  // in `state`
  int backtrack(int sg, int64_t* state, uint8_t* pi, cudaStream_t st) {
    const int k0 = g.seg_begin(sg), cnt = g.seg_begin(sg + 1) - k0;
    int rc = SP_OK;
    if (!separate) {
      for (int p = g.nparts - 1; p >= 0 && !rc; --p) {
        grid_backtrack_part_kernel<<<1, 1, 0, st>>>(g.shifts(pw[p]), g.bp(pw[p]), g.row_words, g.mode, k0, cnt,
                                                    (int64_t)p * g.Wp, state, pi);
        rc = launch_check("grid_backtrack_part_kernel launch");
      }
      return rc;
    }
    rc = check_cuda(cudaEventRecord(start, st), "record backtrack start");
    cudaEvent_t prev = start;
    for (int p = g.nparts - 1; p >= 0 && !rc; --p) {
      cudaSetDevice(dev[p]);
      rc = check_cuda(cudaStreamWaitEvent(pst[p], prev, 0), "backtrack handoff wait");
      if (rc) break;
      grid_backtrack_part_kernel<<<1, 1, 0, pst[p]>>>(g.shifts(pw[p]), g.bp(pw[p]), g.row_words, g.mode, k0, cnt,
                                                      (int64_t)p * g.Wp, state, pi);
      rc = launch_check("grid_backtrack_part_kernel launch");
      if (!rc) rc = check_cuda(cudaEventRecord(ev[p], pst[p]), "record handoff");
      prev = ev[p];
    }
    cudaSetDevice(cur);
    if (!rc) rc = check_cuda(cudaStreamWaitEvent(st, prev, 0), "join backtrack");
    return rc;
  }
};

// Devices and partition workspaces of an sp_plan_dp_devices call.
struct DevPlan {
  int n = 0;
  int dev[kMaxParts] = {};
  uint8_t* ws[kMaxParts] = {};
  size_t bytes[kMaxParts] = {};
};

int read_max_shift(const StageShift* shifts, int L, cudaStream_t st, int* ms) {
  std::vector<StageShift> hs(L);
  int rc = check_cuda(cudaMemcpyAsync(hs.data(), shifts, sizeof(StageShift) * L, cudaMemcpyDeviceToHost, st),
                      "copy stage shifts");
  if (!rc) rc = check_cuda(cudaStreamSynchronize(st), "sync");
  int m = 0;
  for (const StageShift& x : hs) m = std::max(m, max_shift(x));
  *ms = m;
  return rc;
}

// Solve one instance over capacity partitions.  With
// every back-pointer stage in memory: one forward launch and one backtrack.
// Otherwise checkpoint / recompute: a forward pass keeping a checkpoint row
// at every segment boundary (segments aligned to the END of the chain, the
// last keeping its back-pointers from the forward pass), then, segment by
// segment from the end, a recompute of the segment's back-pointers from its
// checkpoint and a backtrack through it: 2L - K stages of DP work.  Every
// partition keeps its rows, checkpoints and back-pointers in its own
// workspace; the backtrack walks partition by partition from the right,
// handing (stage, column, side) leftwards.
// `dp` (sp_plan_dp_devices): one partition per listed device, each in the
// caller's workspace for it; otherwise SPLITPLAN_GRID_PARTS partitions (1 by
// default) carved from `dyn` on this device.
int run_grid_instance(const sp_instances* in, sp_policies* out, InstInfo* info, const StageShift* shifts,
                      const int64_t* rv, const int2* reach, int32_t* idx, int64_t* gstate, int64_t inst, int64_t lo,
                      int L, int64_t ncol, int mode, uint8_t* dyn, size_t avail, cudaStream_t st,
                      const DevPlan* dp) {
  GridRun R;
  cudaGetDevice(&R.cur);
  int nparts = dp ? dp->n : std::max(1, std::min(kMaxParts, env_int("SPLITPLAN_GRID_PARTS", 1)));
  int ms = 0;
  int rc = SP_OK;
  if (nparts > 1) {
    rc = read_max_shift(shifts + lo, L, st, &ms);
    if (rc) return rc;
  }
  const int resident = grid_resident_rt(mode);
  if (resident <= 0) return check_cuda(cudaErrorInvalidConfiguration, "dp_grid_kernel occupancy");
  const int force_k = env_int("SPLITPLAN_GRID_SEGMENT", 0);
  GridGeom g;
  for (;;) {
    // CTAs per partition: every partition placed on one device must be co-resident there
    int per_dev = dp ? 1 : nparts;
    size_t part_avail = dp ? dp->bytes[0] : avail / (size_t)nparts;
    if (dp) {
      for (int p = 0; p < nparts; ++p) {
        int c = 0;
        for (int r = 0; r < nparts; ++r) c += dp->dev[r] == dp->dev[p];
        per_dev = std::max(per_dev, c);
        part_avail = std::min(part_avail, dp->bytes[p]);
      }
    }
    part_avail = part_avail / 256 * 256;
    bool too_wide = false;
    rc = grid_geometry(mode, L, ncol, nparts, resident / per_dev, ms, part_avail, force_k, &g, &too_wide);
    if (!dp && !too_wide && g.nparts < nparts) {  // fewer chunks than partitions: re-split dyn
      nparts = g.nparts;
      continue;
    }
    if (rc == SP_ERR_WORKSPACE && !dp)  // every partition is carved from dyn
      set_required_workspace((size_t)g.nparts * g.part_bytes);
    if (rc) return rc;
    if (!too_wide) break;
    nparts = 1;  // the read-back spans a whole partition: no point splitting
  }
  R.g = g;
  const bool dev_list = dp != nullptr;
  for (int p = 0; p < g.nparts; ++p) {
    R.dev[p] = dev_list ? dp->dev[p] : R.cur;
    R.pw[p] = dev_list ? dp->ws[p] : dyn + (size_t)p * g.part_bytes;
    if (R.dev[p] != R.cur) R.multi = true;
  }
  R.separate = g.nparts > 1 && (dev_list || env_int("SPLITPLAN_GRID_SEPARATE", 0) != 0);
  R.sys = (dev_list || env_int("SPLITPLAN_GRID_SYS", 0)) ? 1 : 0;
  R.use_reach = reach != nullptr;
  if (R.multi) {  // every used device reaches every other one
    for (int p = 0; p < g.nparts; ++p)
      for (int r = 0; r < g.nparts; ++r) {
        if (R.dev[p] == R.dev[r]) continue;
        cudaSetDevice(R.dev[p]);
        const cudaError_t e = cudaDeviceEnablePeerAccess(R.dev[r], 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
          cudaSetDevice(R.cur);
          return check_cuda(e, "cudaDeviceEnablePeerAccess");
        }
        cudaGetLastError();
      }
    cudaSetDevice(R.cur);
  }
  if (R.separate) {
    rc = R.init_streams();
    if (rc) return rc;
  }
  // every partition gets its own copy of the stage records
  for (int p = 0; p < g.nparts && !rc; ++p) {
    rc = check_cuda(cudaMemcpyAsync(g.shifts(R.pw[p]), shifts + lo, sizeof(StageShift) * L, cudaMemcpyDefault, st),
                    "copy stage shifts to partition");
    if (!rc)
      rc = check_cuda(cudaMemcpyAsync(g.rv(R.pw[p]), rv + lo, sizeof(int64_t) * L, cudaMemcpyDefault, st),
                      "copy stage values to partition");
    if (!rc && reach)
      rc = check_cuda(cudaMemcpyAsync(g.reach(R.pw[p]), reach + lo, sizeof(int2) * L, cudaMemcpyDefault, st),
                      "copy frontiers to partition");
  }
  if (rc) return rc;
  {
    uint8_t sac = 0;
    rc = check_cuda(cudaMemcpyAsync(&sac, in->source_at_client + inst, 1, cudaMemcpyDeviceToHost, st),
                    "copy source_at_client");
    if (!rc) rc = check_cuda(cudaStreamSynchronize(st), "sync");
    if (rc) return rc;
    R.g.sac = sac ? 1 : 0;
  }
  const GridGeom& G = R.g;
  auto timed_phase = [&](int k0, int cnt, int init_ckpt, int out_ckpt, bool keep_bp) -> int {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (profiling()) {
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, st);
    }
    int r = R.phase(k0, cnt, init_ckpt, out_ckpt, keep_bp, st);
    if (r) return r;
    if (profiling()) {
      cudaEventRecord(e1, st);
      const double cells = (double)cnt * (double)ncol;
      prof_record_dp(e0, e1, cells, cells * (keep_bp ? hbm_bytes_per_cell(mode, DPV_SMEM) : 0.0), DPV_GRID);
    }
    return SP_OK;
  };
  // forward pass
  for (int sg = 0; sg < G.nseg && !rc; ++sg) {
    const int k0 = G.seg_begin(sg), cnt = G.seg_begin(sg + 1) - k0;
    rc = timed_phase(k0, cnt, sg, sg + 1, sg + 1 == G.nseg);
  }
  if (rc) return rc;
  const int own = G.owner_part();
  grid_end_kernel<<<1, 1, 0, st>>>(info + inst, (int64_t)own * G.Wp, G.Wp, L, -1,
                                   in->must_end_at ? in->must_end_at + inst : nullptr, G.ckpt(R.pw[own], G.nseg),
                                   gstate);
  rc = launch_check("grid_end_kernel launch");
  if (rc || !out) return rc;
  for (int sg = G.nseg - 1; sg >= 0 && !rc; --sg) {
    if (sg + 1 < G.nseg) {  // the last segment's back-pointers are still there
      const int k0 = G.seg_begin(sg), cnt = G.seg_begin(sg + 1) - k0;
      rc = timed_phase(k0, cnt, sg, 0, true);
    }
    if (!rc) rc = R.backtrack(sg, gstate, out->pi + lo, st);
  }
  if (rc) return rc;
  grid_finish_kernel<<<1, 1, 0, st>>>(*in, inst, gstate, idx, *out);
  return launch_check("grid_finish_kernel launch");
  // the caller's next use of the workspace is stream-ordered after these
}

// Workspace of the whole-GPU path for one instance in one partition on this
// device: the smallest that runs it (checkpoint / recompute) and the one that
// keeps every back-pointer stage.
void grid_workspace_bytes(int mode, int64_t L, int64_t ncol, int nparts, int per_dev, int max_shift,
                          size_t* min_bytes, size_t* full_bytes) {
  GridGeom g;
  bool too_wide = false;
  const int resident = std::max(1, grid_resident_rt(mode));
  const size_t huge = ~(size_t)0 >> 2;
  grid_geometry(mode, (int)L, ncol, nparts, resident / std::max(per_dev, 1), max_shift, huge, 0, &g, &too_wide);
  if (too_wide) grid_geometry(mode, (int)L, ncol, 1, resident, max_shift, huge, 0, &g, &too_wide);
  *full_bytes = g.part_bytes;
  GridGeom t = g;
  grid_layout(t, 1);
  int kopt = (int)std::max(1.0, std::sqrt((double)L * (double)t.ckpt_bytes / (double)t.bp_stage));
  kopt = (int)std::min<int64_t>(kopt, L);
  grid_layout(t, kopt);
  *min_bytes = std::min(t.part_bytes, g.part_bytes);
  const int force_k = env_int("SPLITPLAN_GRID_SEGMENT", 0);
  if (force_k > 0) {  // a forced segment length needs exactly its layout
    grid_layout(t, (int)std::min<int64_t>(force_k, L));
    *min_bytes = *full_bytes = t.part_bytes;
  }
}

// Shared driver of sp_plan_dp and sp_build_dp_tables.
// `dp`: sp_plan_dp_devices' devices and partition workspaces (null: one
// device, partitions in `ws`).  Workspace query (q_min != null): nothing is
// planned; q_min / q_full receive the bytes of `ws` (and q_part_min /
// q_part_full those of each partition workspace when `dp` is set).
// `w_eff_check` >= 0: build_dp_tables' caller-sized tables, checked against
// the instance's W_eff before anything is written.
// Pending state of sp_plan_dp_async / sp_plan_dp_finish, in the caller's
// pinned host buffer of SP_PENDING_BYTES bytes.
struct PendingRec {
  unsigned long long solved[4];  // tier 1's counters, copied there by the stream
  cudaEvent_t ev;                // recorded after that copy
  int32_t mode;                  // 0: nothing pending (the call ran to completion), 1: tier 1 in flight
  int32_t pad;
};
static_assert(sizeof(PendingRec) <= SP_PENDING_BYTES, "pending record");

// `begin`: enqueue tier 1 and return (its counters land in begin->solved);
// `resume`: the second half of such a call -- nothing is launched again, the
// counters are waited for and the host-planned tiers run for what is left.
int run_dp(const sp_instances* in, sp_policies* out, double* tab_c, double* tab_s, void* ws,
           size_t ws_bytes, cudaStream_t st, size_t* q_min = nullptr, size_t* q_full = nullptr,
           const DevPlan* dp = nullptr, size_t* q_part_min = nullptr, size_t* q_part_full = nullptr,
           int64_t w_eff_check = -1, PendingRec* begin = nullptr, PendingRec* resume = nullptr) {
  const int64_t n = in->n, total = in->total_layers;
  if (n == 0) return SP_OK;
  const Trace trace;
  trace("run_dp begin", n);
  if (ws && ((uintptr_t)ws & 255)) {
    set_error(SP_ERR_INVALID, "workspace must be 256-byte aligned (cudaMalloc alignment)");
    return SP_ERR_INVALID;
  }
  Carve cv{(uint8_t*)ws, ws_bytes};
  InstInfo* info = (InstInfo*)cv.take(sizeof(InstInfo) * n);
  StageShift* shifts = (StageShift*)cv.take(sizeof(StageShift) * total);
  int64_t* rv = (int64_t*)cv.take(sizeof(int64_t) * total);
  int32_t* idx = (int32_t*)cv.take(sizeof(int32_t) * total);
  DpWork* work = (DpWork*)cv.take(sizeof(DpWork) * n);
  int2* reach = (int2*)cv.take(sizeof(int2) * total);
  int64_t* gstate = (int64_t*)cv.take(64);
  int32_t* overflow = (int32_t*)cv.take(sizeof(int32_t) * n);
  int32_t* flag = (int32_t*)cv.take(sizeof(int32_t) * n);
  unsigned long long* solved = (unsigned long long*)cv.take(4 * sizeof(unsigned long long));
  const int64_t t0_nblk = (n + kT0Block - 1) / kT0Block;
  T0Stats* t0s = (T0Stats*)cv.take(sizeof(T0Stats));
  T0Block* t0blk = (T0Block*)cv.take(sizeof(T0Block) * t0_nblk);
  uint8_t* t0cls = (uint8_t*)cv.take(n);
  const size_t fixed = align_up(cv.used, 256);
  if (!ws || fixed > ws_bytes) {
    set_required_workspace(fixed + (1 << 20));
    set_full_workspace(fixed + (1 << 20));  // unknown until the prep kernel has run
    set_error(SP_ERR_WORKSPACE, "workspace %zu B < fixed part %zu B", ws_bytes, fixed);
    return SP_ERR_WORKSPACE;
  }
  const int force = forced_variant();
  const bool steps_allowed = tab_c == nullptr && (force < 0 || force == DPV_STEPS);
  const bool steps_ok = steps_allowed && !q_min;
  const int grid = (int)std::min<int64_t>((n + kPrepWarps - 1) / kPrepWarps, 1 << 20);
  // tier 1 in one launch when every instance's store fits the workspace, else
  // (not in an asynchronous call) in waves of consecutive instances
  const size_t rpb = steps_row_pair_bytes(kStepsCap);
  const bool tier1_one = steps_ok && out && fixed + (size_t)(total + n) * rpb <= ws_bytes;
  const bool tier1_fits = tier1_one || (steps_ok && out && !begin && !resume && fixed + 64 * rpb <= ws_bytes &&
                                        env_int("SPLITPLAN_NO_TIER1_WAVES", 0) == 0);
  const int64_t lo_i32 = steps_min_cols(VM_INT32, force), lo_f64 = steps_min_cols(VM_F64, force);
  // tier 0 (the SMEM kernel's instances, planned on the device): the default
  // kernel choice only (no forced variant or configuration), not for the
  // workspace query, full tables, or the first half of an asynchronous call
  // (the workspace query counts its instances the same way, to size it)
  const bool t0_allowed = (out || q_min) && tab_c == nullptr && force < 0 && !getenv("SPLITPLAN_DP_THREADS") &&
                          !getenv("SPLITPLAN_DP_SINGLE_E") && env_int("SPLITPLAN_NO_TIER0", 0) == 0;
  const bool t0_count = t0_allowed && !begin;  // classify and count
  const bool t0_ok = t0_count && !q_min;        // and run
  int rc = SP_OK;
  if (!resume) {
    prep_kernel<<<grid, 128, 0, st>>>(*in, info, shifts, rv, reach, (steps_ok || t0_allowed) ? flag : nullptr,
                                      tier1_fits ? kGridMinColsSteps : 0, lo_i32, lo_f64);
    rc = launch_check("prep_kernel launch");
    if (rc) return rc;
  }
  uint8_t* dyn = (uint8_t*)ws + fixed;
  // tier-0 classification and counts, queued after tier 1 (the instances it
  // left keep their flag); the totals travel with the next synchronisation
  bool t0_counted = false;
  auto launch_t0_count = [&]() -> int {
    if (!t0_count || t0_counted) return SP_OK;
    t0_counted = true;
    int r = check_cuda(cudaMemsetAsync(t0s, 0, sizeof(T0Stats), st), "zero tier-0 counters");
    if (r) return r;
    T0Skip skip = {{0, 0, 0}};
    if (q_min && steps_allowed) skip = T0Skip{{lo_i32, lo_f64, kGridMinColsSteps}};
    t0_count_kernel<<<(unsigned)t0_nblk, kT0Block, 0, st>>>(*in, info, (steps_ok || t0_allowed) ? flag : nullptr,
                                                           smem_max_cols(VM_INT32), smem_max_cols(VM_F64), skip,
                                                           t0cls, t0s, t0blk);
    return launch_check("t0_count_kernel launch");
  };
  T0Stats ht0 = {};
  std::vector<T0Block> hblk;
  bool ht0_valid = false;
  auto copy_t0 = [&]() -> int {  // queue the tier-0 counts' copy (the caller synchronises)
    hblk.resize((size_t)t0_nblk);
    int r = check_cuda(cudaMemcpyAsync(&ht0, t0s, sizeof(T0Stats), cudaMemcpyDeviceToHost, st), "copy tier-0 max");
    if (!r)
      r = check_cuda(cudaMemcpyAsync(hblk.data(), t0blk, sizeof(T0Block) * t0_nblk, cudaMemcpyDeviceToHost, st),
                     "copy tier-0 counts");
    ht0_valid = true;
    return r;
  };

  // Tier 1, planned on the device: one warp per instance on breakpoint lists
  // of kStepsCap breakpoints, every store at a position the kernel computes
  // itself -- no host planning, one synchronisation for the whole batch.
  // Instances it cannot take (NaN domain, whole-GPU width, more breakpoints)
  // keep their flag and go through the host-planned tiers below.
  bool tier1 = false;
  unsigned long long tier1_solved = 0;
  if (tier1_fits) {
    tier1 = true;
    StepsArgs sa = {};
    sa.layer_off = in->layer_off;
    sa.sac = in->source_at_client;
    sa.info = info;
    sa.shifts = shifts;
    sa.rv = rv;
    sa.store = dyn;
    sa.flag = flag;
    sa.solved = solved;
    sa.n_items = n;
    sa.max_cols = kGridMinColsSteps;
    sa.min_cols[0] = lo_i32;
    sa.min_cols[1] = lo_f64;
    unsigned long long hsolved[4] = {0, 0, 0, 0};  // instances, DP cells, breakpoints, stages
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (resume) {
      rc = check_cuda(cudaEventSynchronize(resume->ev), "wait for tier 1");
      cudaEventDestroy(resume->ev);
      resume->ev = nullptr;
      resume->mode = 0;
      if (rc) return rc;
      memcpy(hsolved, resume->solved, sizeof(hsolved));
    } else {
      rc = check_cuda(cudaMemsetAsync(solved, 0, 4 * sizeof(unsigned long long), st), "zero solved count");
      if (!rc && profiling() && !begin) {
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, st);
      }
      if (tier1_one) {
        sa.item0 = 0;
        sa.pos0 = 0;
        if (!rc) rc = launch_steps(VM_INT32, kStepsCap, sa, in, out, idx, st);
        if (!rc) rc = launch_steps(VM_F64, kStepsCap, sa, in, out, idx, st);
      } else if (!rc) {
        // waves: consecutive instances whose stores fit (an instance alone too
        // large for the workspace keeps its flag for the next tiers)
        std::vector<int64_t> ho(n + 1);
        rc = check_cuda(cudaMemcpyAsync(ho.data(), in->layer_off, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost,
                                        st),
                        "copy layer offsets");
        if (!rc) rc = check_cuda(cudaStreamSynchronize(st), "sync for tier-1 waves");
        const size_t avail1 = ws_bytes - fixed;
        int64_t i0 = 0;
        while (!rc && i0 < n) {
          int64_t i1 = i0;
          while (i1 < n && (size_t)(ho[i1 + 1] - ho[i0] + (i1 + 1 - i0)) * rpb <= avail1) ++i1;
          if (i1 == i0) {
            ++i0;
            continue;
          }
          sa.item0 = i0;
          sa.pos0 = ho[i0] + i0;
          sa.n_items = i1 - i0;
          rc = launch_steps(VM_INT32, kStepsCap, sa, in, out, idx, st);
          if (!rc) rc = launch_steps(VM_F64, kStepsCap, sa, in, out, idx, st);
          trace("tier-1 wave", (long long)(i1 - i0));
          i0 = i1;
        }
      }
      if (!rc && e1) cudaEventRecord(e1, st);
      if (!rc && begin) {  // asynchronous: the counters travel to the caller's pinned buffer
        rc = check_cuda(cudaMemcpyAsync(begin->solved, solved, sizeof(hsolved), cudaMemcpyDeviceToHost, st),
                        "copy solved count");
        if (!rc) rc = check_cuda(cudaEventCreateWithFlags(&begin->ev, cudaEventDisableTiming), "event");
        if (!rc) rc = check_cuda(cudaEventRecord(begin->ev, st), "record tier 1");
        if (!rc) begin->mode = 1;
        return rc;
      }
      if (!rc)
        rc = check_cuda(cudaMemcpyAsync(hsolved, solved, sizeof(hsolved), cudaMemcpyDeviceToHost, st),
                        "copy solved count");
      if (!rc) rc = launch_t0_count();
      if (!rc && t0_ok) rc = copy_t0();
      if (!rc) rc = check_cuda(cudaStreamSynchronize(st), "sync after breakpoint lists");
      if (rc) return rc;
    }
    // algorithmic HBM bytes of the breakpoint-list kernel: the stage records it
    // reads (16 B shifts + 8 B value per stage) and the store it writes (an
    // 8-B {column, stay_from} per breakpoint, a 4-B count per row)
    if (e1)
      prof_record_dp(e0, e1, (double)hsolved[1],
                     24.0 * (double)hsolved[3] + 8.0 * (double)hsolved[2] +
                         8.0 * (double)(hsolved[3] + hsolved[0]),
                     DPV_STEPS);
    tier1_solved = hsolved[0];
  }

  // Tier 0: every instance of the SMEM kernel's range, in waves of whole
  // counting blocks whose back-pointer tables fit after tier 1's store
  unsigned long long t0_taken = 0;
  size_t t0_peak = 0;
  // (tier 1's stores are dead once its kernels are: their walk is fused)
  const size_t region0 = 0;
  std::vector<uint8_t> hcls;  // the query: tier-0 classes (255: a host-planned tier's instance)
  if (t0_count && !ht0_valid && tier1_solved < (unsigned long long)n) {
    rc = launch_t0_count();
    if (!rc) rc = copy_t0();
    if (!rc && q_min) {
      hcls.resize(n);
      rc = check_cuda(cudaMemcpyAsync(hcls.data(), t0cls, n, cudaMemcpyDeviceToHost, st), "copy tier-0 classes");
    }
    if (!rc) rc = check_cuda(cudaStreamSynchronize(st), "sync after tier-0 count");
    if (rc) return rc;
  }
  if (t0_ok && ht0_valid) {
    uint8_t* base0 = dyn + region0;
    const size_t avail0 = ws_bytes > fixed + region0 ? ws_bytes - fixed - region0 : 0;
    bool fits = true;
    unsigned long long cnt = 0;
    for (const T0Block& b : hblk) {
      fits &= b.bytes <= avail0;
      for (int c = 0; c < kT0Classes; ++c) cnt += b.count[c];
    }
    if (cnt > 0 && fits) {
      DpArgs a0 = {};
      a0.layer_off = in->layer_off;
      a0.sac = in->source_at_client;
      a0.info = info;
      a0.shifts = shifts;
      a0.rv = rv;
      a0.bp = base0;
      a0.rows = base0;
      int64_t b_lo = 0;
      while (b_lo < t0_nblk) {
        // one wave: whole blocks while their tables fit
        int64_t b_hi = b_lo;
        size_t wbytes = 0;
        unsigned long long wcnt[kT0Classes] = {}, wcells[kT0Classes] = {};
        while (b_hi < t0_nblk && wbytes + hblk[b_hi].bytes <= avail0) {
          wbytes += hblk[b_hi].bytes;
          for (int c = 0; c < kT0Classes; ++c) {
            wcnt[c] += hblk[b_hi].count[c];
            wcells[c] += hblk[b_hi].cells[c];
          }
          ++b_hi;
        }
        T0Seg seg;
        unsigned long long acc = 0;
        for (int c = 0; c < kT0Classes; ++c) {
          seg.off[c] = acc;
          acc += wcnt[c];
        }
        t0_peak = std::max(t0_peak, wbytes);
        if (acc) {
          rc = check_cuda(cudaMemsetAsync(&t0s->cursor, 0, sizeof(unsigned long long) * (kT0Classes + 1), st),
                          "zero tier-0 cursors");
          if (rc) return rc;
          t0_scatter_kernel<<<(unsigned)(b_hi - b_lo), kT0Block, 0, st>>>(*in, info, t0cls, b_lo, seg, t0s, work,
                                                                          flag);
          rc = launch_check("t0_scatter_kernel launch");
          if (rc) return rc;
          for (int c = 0; c < kT0Classes; ++c) {
            const unsigned long long m = wcnt[c];
            if (!m) continue;
            const int mode = t0_class_mode(c), cfg = t0_class_cfg(c);
            DpArgs ga = a0;
            ga.work = work + seg.off[c];
            const size_t smem = stage_bytes_mode(mode) + single_row_bytes(mode, (int64_t)ht0.max_ncol[c], cfg);
            cudaEvent_t e0 = nullptr, e1 = nullptr;
            if (profiling()) {
              cudaEventCreate(&e0);
              cudaEventCreate(&e1);
              cudaEventRecord(e0, st);
            }
            switch (mode) {
              case VM_INT32: rc = launch_single<VM_INT32, true>(ga, (int64_t)m, cfg, smem, st); break;
              case VM_F64: rc = launch_single<VM_F64, true>(ga, (int64_t)m, cfg, smem, st); break;
              default: rc = launch_single<VM_F64_NAN, true>(ga, (int64_t)m, cfg, smem, st); break;
            }
            if (rc) return rc;
            if (profiling()) {
              cudaEventRecord(e1, st);
              prof_record_dp(e0, e1, (double)wcells[c], (double)wcells[c] * hbm_bytes_per_cell(mode, DPV_SMEM),
                             DPV_SMEM);
            }
            backtrack_kernel<<<(unsigned)((m + 127) / 128), 128, 0, st>>>(*in, info, shifts, work + seg.off[c],
                                                                          (int64_t)m, base0, idx, *out);
            rc = launch_check("backtrack_kernel launch");
            if (rc) return rc;
          }
        }
        trace("tier-0 wave", (long long)acc);
        b_lo = b_hi;
      }
      t0_taken = cnt;
    }
  }
  if (q_min && !hcls.empty()) {  // the query, every instance in tier 0: no host planning
    unsigned long long cnt = 0, all = 0, mx = 0;
    for (const T0Block& b : hblk) {
      for (int c = 0; c < kT0Classes; ++c) cnt += b.count[c];
      all += b.bytes;
      mx = std::max(mx, b.bytes);
    }
    if (cnt == (unsigned long long)n) {
      *q_min = fixed + (size_t)mx;
      *q_full = fixed + (size_t)all;
      if (q_part_min) *q_part_min = 0;
      if (q_part_full) *q_part_full = 0;
      return SP_OK;
    }
  }
  if (tier1_solved + t0_taken == (unsigned long long)n) {
    unsigned long long t0_all = 0;
    for (const T0Block& b : hblk) t0_all += b.bytes;
    set_full_workspace(fixed + std::max((size_t)t0_all, tier1 ? (size_t)(total + n) * rpb : (size_t)0));
    set_steps_overflow(0);
    return SP_OK;
  }

  std::vector<InstInfo> hinfo(n);
  std::vector<int64_t> hoff(n + 1);
  rc = check_cuda(cudaMemcpyAsync(hinfo.data(), info, sizeof(InstInfo) * n, cudaMemcpyDeviceToHost, st),
                  "copy instance info");
  if (rc) return rc;
  rc = check_cuda(cudaMemcpyAsync(hoff.data(), in->layer_off, sizeof(int64_t) * (n + 1),
                                  cudaMemcpyDeviceToHost, st),
                  "copy layer offsets");
  if (rc) return rc;
  rc = check_cuda(cudaStreamSynchronize(st), "sync after prep");
  if (rc) return rc;
  trace("prep done, info on host");

  if (w_eff_check >= 0 && hinfo[0].w_eff != w_eff_check) {
    set_error(SP_ERR_INVALID, "w_eff = %lld does not match the instance's effective budget %lld",
              (long long)w_eff_check, (long long)hinfo[0].w_eff);
    return SP_ERR_INVALID;
  }
  const size_t avail = ws_bytes - fixed;
  std::vector<int32_t> hflag;
  if (tier1 || t0_taken) {  // the instances tiers 1 and 0 left: the next tiers take only them
    hflag.resize(n);
    rc = check_cuda(cudaMemcpyAsync(hflag.data(), flag, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st),
                    "copy tier-1 flags");
    if (!rc) rc = check_cuda(cudaStreamSynchronize(st), "sync");
    if (rc) return rc;
  }
  struct Item {
    int64_t inst, L, ncol;
    int mode;
    DpPlan plan;
  };
  std::vector<Item> items;
  items.reserve(n);
  DpPlan cached;
  int cached_mode = -1;
  int64_t cached_ncol = -1, cached_L = -1;
  int cached_cap = -1;
  // the query's tier-1 instances are sized in O(1) each: their stores summed,
  // the dense fallback's minimum bounded by the widest and longest per domain
  // (both monotone in L and W_eff), instead of a launch plan per instance
  size_t q_tier1 = 0;
  int64_t q_maxL[3] = {0, 0, 0}, q_maxcol[3] = {0, 0, 0};
  for (int64_t k = 0; k < n; ++k) {
    if (!hflag.empty() && !hflag[k]) continue;  // solved by tier 1 (breakpoint lists) or tier 0
    if (!hcls.empty() && hcls[k] != 255) continue;  // the query: tier 0's (sized below)
    const int64_t ncol = hinfo[k].w_eff + 1;
    if (ncol > kMaxCols) {
      set_error(SP_ERR_UNSUPPORTED, "instance %lld: W_eff = %lld exceeds the supported 2^31 columns",
                (long long)k, (long long)hinfo[k].w_eff);
      return SP_ERR_UNSUPPORTED;
    }
    if (q_min && steps_allowed && ncol < kGridMinCols && force != DPV_GRID &&
        steps_eligible(hinfo[k].mode, ncol, force, false, lo_i32, lo_f64)) {
      const int64_t L = hoff[k + 1] - hoff[k];
      const int m = hinfo[k].mode;
      q_tier1 += (size_t)(L + 1) * rpb;
      q_maxL[m] = std::max(q_maxL[m], L);
      q_maxcol[m] = std::max(q_maxcol[m], ncol);
      continue;
    }
    Item it;
    it.inst = k;
    it.L = hoff[k + 1] - hoff[k];
    it.ncol = ncol;
    it.mode = hinfo[k].mode;
    // breakpoint lists first (tier 1 if it did not run, else the wide tier)
    // (a tier whose store does not fit the workspace is skipped: the tiers are
    // an optimisation, the dense kernels the guarantee)
    int cap = steps_ok && steps_eligible(it.mode, ncol, force, tab_c != nullptr, lo_i32, lo_f64)
                  ? (tier1 ? kStepsCapWide : kStepsCap)
                  : 0;
    if (cap == kStepsCap && align_up(steps_store_bytes((int)it.L, cap), 256) > avail) cap = kStepsCapWide;
    if (cap == kStepsCapWide && align_up(steps_store_bytes((int)it.L, cap), 256) > avail) cap = 0;
    if (it.mode != cached_mode || ncol != cached_ncol || it.L != cached_L || cap != cached_cap) {
      cached = plan_instance(it.mode, it.L, ncol, force, tab_c != nullptr, cap);
      cached_mode = it.mode;
      cached_ncol = ncol;
      cached_L = it.L;
      cached_cap = cap;
    }
    it.plan = cached;
    items.push_back(it);
  }

  if (q_min) {  // workspace query: no DP launched
    size_t mn = 0, full = 0, pmn = 0, pfull = 0;
    const int nparts = dp ? dp->n : std::max(1, std::min(kMaxParts, env_int("SPLITPLAN_GRID_PARTS", 1)));
    int per_dev = dp ? 1 : nparts;
    if (dp)
      for (int p = 0; p < dp->n; ++p) {
        int c = 0;
        for (int r = 0; r < dp->n; ++r) c += dp->dev[r] == dp->dev[p];
        per_dev = std::max(per_dev, c);
      }
    size_t tier1 = 0;  // the device-planned breakpoint lists' store of the eligible instances
    for (const Item& it : items) {
      const bool grid = tab_c == nullptr && (force == DPV_GRID || it.ncol >= kGridMinCols);
      size_t imin = it.plan.bp + it.plan.rows, ifull = imin;
      if (!grid && steps_allowed && steps_eligible(it.mode, it.ncol, force, false, lo_i32, lo_f64)) {
        // the minimum stays the dense kernels' (every instance may fall back
        // to them); the useful size is the breakpoint store
        mn = std::max(mn, imin);
        tier1 += (size_t)(it.L + 1) * steps_row_pair_bytes(kStepsCap);
        continue;
      }
      if (grid) {
        int ms = 0;
        if (nparts > 1) {
          rc = read_max_shift(shifts + hoff[it.inst], (int)it.L, st, &ms);
          if (rc) return rc;
        }
        grid_workspace_bytes(it.mode, it.L, it.ncol, nparts, per_dev, ms, &imin, &ifull);
        if (dp) {  // partitions live in their own workspaces
          pmn = std::max(pmn, imin);
          pfull = std::max(pfull, ifull);
          continue;
        }
        imin *= (size_t)nparts;
        ifull *= (size_t)nparts;
      }
      mn = std::max(mn, imin);
      full = grid ? std::max(full, ifull) : full + ifull;
    }
    tier1 += q_tier1;
    for (int m = 0; m < 3; ++m)
      if (q_maxL[m] > 0) {  // the dense kernels' need of any tier-1 instance that overflows
        const DpPlan p = plan_instance(m, q_maxL[m], q_maxcol[m], force, false, 0);
        mn = std::max(mn, p.bp + p.rows);
      }
    size_t t0_all = 0;  // tier 0: its tables in one wave (useful), one counting block's (minimum)
    for (const T0Block& b : hblk) {
      t0_all += b.bytes;
      mn = std::max(mn, (size_t)b.bytes);
    }
    *q_min = fixed + mn;
    *q_full = fixed + std::max(std::max(full, tier1), std::max((size_t)t0_all, mn));
    if (q_part_min) *q_part_min = pmn;
    if (q_part_full) *q_part_full = pfull;
    return SP_OK;
  }
  const int2* a_reach = env_int("SPLITPLAN_NO_REACH", 0) ? nullptr : reach;
  // instances too large for a wave (or wider than 4M columns) run alone over
  // the whole GPU (grid path, checkpointing if needed)
  // The workspace that would run every wave-path instance in ONE wave and
  // keep every back-pointer stage of the whole-GPU ones (reported whether or
  // not this call succeeds: sp_last_full_workspace, so a caller growing its
  // workspace after SP_ERR_WORKSPACE can grow straight to a useful size).
  trace("items planned", (long long)items.size());
  auto is_grid = [&](const Item& it) {
    return tab_c == nullptr && (force == DPV_GRID || it.ncol >= kGridMinCols || it.plan.bp + it.plan.rows > avail);
  };
  {
    size_t one = fixed, grid_full = 0;
    for (const Item& it : items) {
      if (!is_grid(it)) {
        one += it.plan.bp + it.plan.rows;
        continue;
      }
      if (dp) continue;  // partitions live in their own workspaces
      const int np = std::max(1, std::min(kMaxParts, env_int("SPLITPLAN_GRID_PARTS", 1)));
      int ms = 0;
      if (np > 1) {
        rc = read_max_shift(shifts + hoff[it.inst], (int)it.L, st, &ms);
        if (rc) return rc;
      }
      size_t gmin = 0, gfull = 0;
      grid_workspace_bytes(it.mode, it.L, it.ncol, np, np, ms, &gmin, &gfull);
      grid_full = std::max(grid_full, fixed + (size_t)np * gfull);
    }
    set_full_workspace(std::max(one, grid_full));
  }
  {
    std::vector<Item> rest;
    rest.reserve(items.size());
    for (const Item& it : items) {
      if (!is_grid(it)) {
        rest.push_back(it);
        continue;
      }
      rc = run_grid_instance(in, out, info, shifts, rv, a_reach, idx, gstate, it.inst, hoff[it.inst], (int)it.L,
                             it.ncol, it.mode, dyn, avail, st, dp);
      if (rc == SP_ERR_WORKSPACE && !dp) set_required_workspace(fixed + sp_last_required_workspace());
      if (rc) return rc;
    }
    items.swap(rest);
  }

  DpArgs a;
  a.layer_off = in->layer_off;
  a.sac = in->source_at_client;
  a.info = info;
  a.shifts = shifts;
  a.reach = a_reach;
  a.rv = rv;
  a.work = work;
  a.bp = dyn;
  a.rows = dyn;
  a.tab_c = tab_c;
  a.tab_s = tab_s;
  a.overflow = overflow;

  std::vector<DpWork> hwork;
  struct Group {
    int mode;
    DpPlan plan;
    double cells = 0;
    std::vector<DpWork> items;
  };
  std::vector<Group> groups;
  auto run_waves = [&](const std::vector<Item>& items) -> int {
  size_t pos = 0;
  while (pos < items.size()) {
    trace("wave begin", (long long)pos);
    // gather one wave that fits the workspace
    size_t end = pos, wave_bytes = 0;
    while (end < items.size() && wave_bytes + items[end].plan.bp + items[end].plan.rows <= avail) {
      wave_bytes += items[end].plan.bp + items[end].plan.rows;
      ++end;
    }
    if (end == pos) {
      set_required_workspace(fixed + items[pos].plan.bp + items[pos].plan.rows);
      set_error(SP_ERR_WORKSPACE, "instance %lld needs %zu B of DP workspace, %zu B available",
                (long long)items[pos].inst, items[pos].plan.bp + items[pos].plan.rows, avail);
      return SP_ERR_WORKSPACE;
    }
    // lay out the wave (back-pointers, then global rows) grouped by launch
    hwork.clear();
    groups.clear();
    size_t off = 0;
    for (size_t q = pos; q < end; ++q) {
      const Item& it = items[q];
      DpWork w;
      w.inst = it.inst;
      w.bp_off = (int64_t)off;
      w.bp_row_words = it.plan.bp_row_words;
      off += it.plan.bp;
      if (it.plan.rows) {
        w.row_off = (int64_t)off;
        off += it.plan.rows;
      } else {
        w.row_off = -1;
      }
      Group* g = nullptr;
      for (Group& c : groups)
        if (c.mode == it.mode && c.plan.same_launch(it.plan)) g = &c;
      if (!g) {
        groups.push_back(Group{it.mode, it.plan});
        g = &groups.back();
      }
      g->plan.smem = std::max(g->plan.smem, it.plan.smem);
      g->items.push_back(w);
      g->cells += (double)it.L * (double)it.ncol;
    }
    for (const Group& g : groups)
      for (const DpWork& w : g.items) hwork.push_back(w);
    trace("wave laid out", (long long)hwork.size());
    rc = check_cuda(cudaMemcpyAsync(work, hwork.data(), sizeof(DpWork) * hwork.size(),
                                    cudaMemcpyHostToDevice, st),
                    "upload work list");
    if (rc) return rc;
    trace("work list uploaded");
    int64_t first = 0;
    for (const Group& g : groups) {
      const int64_t cnt = (int64_t)g.items.size();
      DpArgs ga = a;
      ga.work = work + first;
      cudaEvent_t e0 = nullptr, e1 = nullptr;
      if (profiling()) {
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, st);
      }
      rc = launch_plan(g.mode, g.plan, ga, cnt, st, in, out, idx);
      if (rc) return rc;
      if (profiling()) {
        cudaEventRecord(e1, st);
        prof_record_dp(e0, e1, g.cells, g.cells * hbm_bytes_per_cell(g.mode, g.plan.variant),
                       g.plan.variant);
      }
      first += cnt;
    }
    if (out) {  // K3 per dense group (the breakpoint-list kernel walks its own instances back)
      first = 0;
      for (const Group& g : groups) {
        const int64_t cnt = (int64_t)g.items.size();
        if (g.plan.variant != DPV_STEPS) {
          backtrack_kernel<<<(unsigned)((cnt + 127) / 128), 128, 0, st>>>(*in, info, shifts, work + first, cnt,
                                                                            dyn, idx, *out);
          rc = launch_check("backtrack_kernel launch");
          if (rc) return rc;
        }
        first += cnt;
      }
    }
    // the host work vector is reused next wave: the pageable H2D copy above is
    // synchronous with respect to the host buffer, so reuse is safe.
    pos = end;
  }
  return SP_OK;
  };
  // instances whose rows outgrew the breakpoint lists move up a tier:
  // kStepsCap -> kStepsCapWide -> the dense kernels
  int64_t dense_fallbacks = 0;
  while (!items.empty()) {
    rc = run_waves(items);
    if (rc) return rc;
    bool any_steps = false;
    for (const Item& it : items) any_steps |= it.plan.variant == DPV_STEPS;
    if (!any_steps) break;
    std::vector<int32_t> hover(n);
    rc = check_cuda(cudaMemcpyAsync(hover.data(), overflow, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st),
                    "copy overflow flags");
    if (!rc) rc = check_cuda(cudaStreamSynchronize(st), "sync overflow flags");
    if (rc) return rc;
    std::vector<Item> redo;
    for (const Item& it : items) {
      if (it.plan.variant != DPV_STEPS || !hover[it.inst]) continue;
      Item r = it;
      int next = it.plan.cfg == kStepsCap ? kStepsCapWide : 0;
      if (next && align_up(steps_store_bytes((int)it.L, next), 256) > avail) next = 0;
      r.plan = plan_instance(it.mode, it.L, it.ncol, force == DPV_STEPS ? -1 : force, false, next);
      dense_fallbacks += next == 0;
      redo.push_back(r);
    }
    items.swap(redo);
  }
  set_steps_overflow(dense_fallbacks);
  trace("run_dp end (launches queued)");
  return SP_OK;
}

}  // namespace
}  // namespace sp

using namespace sp;

extern "C" {

int sp_effective_budget(const sp_instances* in, int64_t* w_eff, void* stream) {
  int rc = validate(in);
  if (rc) return rc;
  if (in->n == 0) return SP_OK;
  if (!w_eff) {
    set_error(SP_ERR_INVALID, "null w_eff");
    return SP_ERR_INVALID;
  }
  const int grid = (int)std::min<int64_t>(in->n, 1 << 20);
  weff_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(*in, w_eff);
  return launch_check("weff_kernel launch");
}

int sp_plan_dp(const sp_instances* in, sp_policies* out, void* ws, size_t ws_bytes, void* stream) {
  int rc = validate(in);
  if (rc) return rc;
  rc = validate_out(out);
  if (rc) return rc;
  return run_dp(in, out, nullptr, nullptr, ws, ws_bytes, (cudaStream_t)stream);
}

}  // extern "C"

// The host-pointer entry points: both sides' (packed) host arrays copied
// through the front of `ws`, `run(device instances, device policies, rest of
// ws, its bytes, stream)` in between, then a stream synchronisation.
template <typename Run>
static int with_host_copies(const char* what, const sp_instances* in, sp_policies* out, void* ws, size_t ws_bytes,
                            void* stream, Run run) {
  int rc = validate(in);
  if (rc) return rc;
  rc = validate_out(out);
  if (rc) return rc;
  const int64_t n = in->n, T = in->total_layers;
  if (n == 0) return SP_OK;
  struct Field {
    const void* p;
    size_t bytes;
  };
  const Field fin[] = {{in->layer_off, 8 * (size_t)(n + 1)}, {in->client_units, 8 * (size_t)T},
                       {in->server_units, 8 * (size_t)T},   {in->up_units, 8 * (size_t)T},
                       {in->down_units, 8 * (size_t)T},     {in->r, 8 * (size_t)T},
                       {in->budget, 8 * (size_t)n},         {in->source_at_client, (size_t)n},
                       {in->must_end_at, in->must_end_at ? (size_t)n : 0}};
  const Field fout[] = {{out->pi, (size_t)T},         {out->client_value, 8 * (size_t)n},
                        {out->server_load, 8 * (size_t)n}, {out->integer_latency, 8 * (size_t)n},
                        {out->feasible, (size_t)n},   {out->status, 4 * (size_t)n}};
  // each side's fields as one span of host memory (callers pack them): one
  // copy in, one copy out
  auto span = [](const Field* f, int k, uintptr_t& lo, uintptr_t& hi) {
    lo = UINTPTR_MAX;
    hi = 0;
    for (int i = 0; i < k; ++i)
      if (f[i].p && f[i].bytes) {
        lo = std::min(lo, (uintptr_t)f[i].p);
        hi = std::max(hi, (uintptr_t)f[i].p + f[i].bytes);
      }
  };
  uintptr_t ilo, ihi, olo, ohi;
  span(fin, 9, ilo, ihi);
  span(fout, 6, olo, ohi);
  const size_t in_bytes = ihi - ilo, out_bytes = ohi - olo;
  const size_t head = align_up(in_bytes, 256) + align_up(out_bytes, 256);
  if (in_bytes > ((size_t)64 << 20) || out_bytes > ((size_t)64 << 20)) {
    set_error(SP_ERR_UNSUPPORTED, "%s: the host arrays must be packed (spans of %zu / %zu B)", what,
              in_bytes, out_bytes);
    return SP_ERR_UNSUPPORTED;
  }
  if (!ws || ws_bytes < head) {
    set_required_workspace(head + (1 << 20));
    set_error(SP_ERR_WORKSPACE, "%s needs %zu B for the copies", what, head);
    return SP_ERR_WORKSPACE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* din = (uint8_t*)ws;
  uint8_t* dout = din + align_up(in_bytes, 256);
  auto dev = [](const void* p, uintptr_t lo, uint8_t* base) -> void* {
    return p ? (void*)(base + ((uintptr_t)p - lo)) : nullptr;
  };
  rc = check_cuda(cudaMemcpyAsync(din, (const void*)ilo, in_bytes, cudaMemcpyHostToDevice, st), "copy instances in");
  if (!rc) rc = check_cuda(cudaMemsetAsync(dout, 0, out_bytes, st), "zero policies");
  if (rc) return rc;
  sp_instances di = *in;
  di.layer_off = (const int64_t*)dev(in->layer_off, ilo, din);
  di.client_units = (const int64_t*)dev(in->client_units, ilo, din);
  di.server_units = (const int64_t*)dev(in->server_units, ilo, din);
  di.up_units = (const int64_t*)dev(in->up_units, ilo, din);
  di.down_units = (const int64_t*)dev(in->down_units, ilo, din);
  di.r = (const double*)dev(in->r, ilo, din);
  di.budget = (const int64_t*)dev(in->budget, ilo, din);
  di.source_at_client = (const uint8_t*)dev(in->source_at_client, ilo, din);
  di.must_end_at = (const int8_t*)dev(in->must_end_at, ilo, din);
  sp_policies dp_ = *out;
  dp_.pi = (uint8_t*)dev(out->pi, olo, dout);
  dp_.client_value = (double*)dev(out->client_value, olo, dout);
  dp_.server_load = (double*)dev(out->server_load, olo, dout);
  dp_.integer_latency = (int64_t*)dev(out->integer_latency, olo, dout);
  dp_.feasible = (uint8_t*)dev(out->feasible, olo, dout);
  dp_.status = (int32_t*)dev(out->status, olo, dout);
  rc = run(&di, &dp_, (uint8_t*)ws + head, ws_bytes - head, st);
  if (rc == SP_ERR_WORKSPACE) set_required_workspace(head + sp_last_required_workspace());
  if (rc) return rc;
  rc = check_cuda(cudaMemcpyAsync((void*)olo, dout, out_bytes, cudaMemcpyDeviceToHost, st), "copy policies out");
  if (!rc) rc = check_cuda(cudaStreamSynchronize(st), "sync");
  return rc;
}


extern "C" {

int sp_plan_dp_host(const sp_instances* in, sp_policies* out, void* ws, size_t ws_bytes, void* stream) {
  return with_host_copies("sp_plan_dp_host", in, out, ws, ws_bytes, stream,
                          [](const sp_instances* di, sp_policies* dout, void* w, size_t wb, cudaStream_t st) {
                            return run_dp(di, dout, nullptr, nullptr, w, wb, st);
                          });
}

int sp_plan_prefix_host(const sp_instances* in, int32_t which, sp_policies* out, void* ws, size_t ws_bytes,
                        void* stream) {
  return with_host_copies("sp_plan_prefix_host", in, out, ws, ws_bytes, stream,
                          [which](const sp_instances* di, sp_policies* dout, void*, size_t, cudaStream_t st) {
                            return sp_plan_prefix(di, which, dout, st);
                          });
}

int sp_plan_dp_async(const sp_instances* in, sp_policies* out, void* ws, size_t ws_bytes, void* stream,
                     void* pending) {
  int rc = validate(in);
  if (rc) return rc;
  rc = validate_out(out);
  if (rc) return rc;
  if (!pending || ((uintptr_t)pending & 7)) {
    set_error(SP_ERR_INVALID, "sp_plan_dp_async: pending must be an 8-B aligned pinned host buffer");
    return SP_ERR_INVALID;
  }
  PendingRec* p = (PendingRec*)pending;
  memset(p, 0, sizeof(PendingRec));
  // runs to completion (mode stays 0) unless tier 1 took the batch
  return run_dp(in, out, nullptr, nullptr, ws, ws_bytes, (cudaStream_t)stream, nullptr, nullptr, nullptr, nullptr,
                nullptr, -1, p, nullptr);
}

int sp_plan_dp_finish(const sp_instances* in, sp_policies* out, void* ws, size_t ws_bytes, void* stream,
                      void* pending) {
  if (!pending) {
    set_error(SP_ERR_INVALID, "sp_plan_dp_finish: null pending");
    return SP_ERR_INVALID;
  }
  PendingRec* p = (PendingRec*)pending;
  if (p->mode != 1) return SP_OK;  // the async call completed the batch itself
  int rc = validate(in);
  if (!rc) rc = validate_out(out);
  if (rc) {
    cudaEventDestroy(p->ev);
    p->mode = 0;
    return rc;
  }
  return run_dp(in, out, nullptr, nullptr, ws, ws_bytes, (cudaStream_t)stream, nullptr, nullptr, nullptr, nullptr,
                nullptr, -1, nullptr, p);
}

size_t sp_plan_dp_onewave_bytes(int64_t n, int64_t total) {
  if (n <= 0 || total < 0) return 0;
  Carve cv{nullptr, 0};  // run_dp's fixed part, laid out the same way
  cv.take(sizeof(InstInfo) * n);
  cv.take(sizeof(StageShift) * total);
  cv.take(sizeof(int64_t) * total);
  cv.take(sizeof(int32_t) * total);
  cv.take(sizeof(DpWork) * n);
  cv.take(sizeof(int2) * total);
  cv.take(64);
  cv.take(sizeof(int32_t) * n);
  cv.take(sizeof(int32_t) * n);
  cv.take(4 * sizeof(unsigned long long));
  cv.take(sizeof(T0Stats));
  cv.take(sizeof(T0Block) * ((n + kT0Block - 1) / kT0Block));
  cv.take(n);
  return align_up(cv.used, 256) + (size_t)(total + n) * steps_row_pair_bytes(kStepsCap);
}

int sp_plan_dp_workspace_bytes(const sp_instances* in, size_t* min_bytes, size_t* full_bytes, void* ws,
                               size_t ws_bytes, void* stream) {
  int rc = validate(in);
  if (rc) return rc;
  if (!min_bytes || !full_bytes) {
    set_error(SP_ERR_INVALID, "null output");
    return SP_ERR_INVALID;
  }
  *min_bytes = *full_bytes = 0;
  if (in->n == 0) return SP_OK;
  return run_dp(in, nullptr, nullptr, nullptr, ws, ws_bytes, (cudaStream_t)stream, min_bytes, full_bytes);
}

// validate a device list and its partition workspaces into a DevPlan
static int dev_plan(const int32_t* devices, int32_t n_devices, void* const* part_ws, const size_t* part_ws_bytes,
                    bool need_ws, DevPlan* dp) {
  int cur = 0, count = 0;
  if (cudaGetDevice(&cur) != cudaSuccess || cudaGetDeviceCount(&count) != cudaSuccess) {
    cudaGetLastError();
    set_error(SP_ERR_CUDA, "no CUDA device");
    return SP_ERR_CUDA;
  }
  if (!devices || n_devices < 1 || n_devices > kMaxParts || devices[0] != cur) {
    set_error(SP_ERR_INVALID, "devices: 1..%d entries, the first the current device (%d)", kMaxParts, cur);
    return SP_ERR_INVALID;
  }
  dp->n = n_devices;
  for (int p = 0; p < n_devices; ++p) {
    if (devices[p] < 0 || devices[p] >= count) {
      set_error(SP_ERR_INVALID, "devices[%d] = %d: no such device", p, devices[p]);
      return SP_ERR_INVALID;
    }
    dp->dev[p] = devices[p];
    if (!need_ws) continue;
    if (!part_ws || !part_ws_bytes || !part_ws[p]) {
      set_error(SP_ERR_INVALID, "partition %d: null workspace", p);
      return SP_ERR_INVALID;
    }
    dp->ws[p] = (uint8_t*)part_ws[p];
    dp->bytes[p] = part_ws_bytes[p];
  }
  return SP_OK;
}

int sp_plan_dp_devices(const sp_instances* in, sp_policies* out, const int32_t* devices, int32_t n_devices,
                       void* ws, size_t ws_bytes, void* const* part_ws, const size_t* part_ws_bytes,
                       void* stream) {
  int rc = validate(in);
  if (rc) return rc;
  rc = validate_out(out);
  if (rc) return rc;
  DevPlan dp;
  rc = dev_plan(devices, n_devices, part_ws, part_ws_bytes, true, &dp);
  if (rc) return rc;
  return run_dp(in, out, nullptr, nullptr, ws, ws_bytes, (cudaStream_t)stream, nullptr, nullptr, &dp);
}

int sp_plan_dp_devices_workspace_bytes(const sp_instances* in, const int32_t* devices, int32_t n_devices,
                                       size_t* ws_min, size_t* part_min, size_t* part_full, void* ws,
                                       size_t ws_bytes, void* stream) {
  int rc = validate(in);
  if (rc) return rc;
  if (!ws_min || !part_min || !part_full) {
    set_error(SP_ERR_INVALID, "null output");
    return SP_ERR_INVALID;
  }
  *ws_min = *part_min = *part_full = 0;
  if (in->n == 0) return SP_OK;
  DevPlan dp;
  rc = dev_plan(devices, n_devices, nullptr, nullptr, false, &dp);
  if (rc) return rc;
  size_t full = 0;
  return run_dp(in, nullptr, nullptr, nullptr, ws, ws_bytes, (cudaStream_t)stream, ws_min, &full, &dp, part_min,
                part_full);
}

// ---- capacity partitions, one process per device ---------------------------

static GridGeom geom_of(const sp_grid_plan* p) {
  GridGeom g;
  g.mode = p->mode;
  g.L = p->n_layers;
  g.G = p->ctas;
  g.NC = p->chunks_per_cta;
  g.nparts = p->nparts;
  g.K = p->seg_stages;
  g.nseg = p->nseg;
  g.nckpt = p->nckpt;
  g.sac = p->sac;
  g.ncol = p->ncol;
  g.B = p->part_cols / std::max(p->ctas, 1);
  g.Wp = p->part_cols;
  g.halo = p->halo;
  g.span = p->span;
  g.row_words = p->row_words;
  g.rec_off = p->rec_off;
  g.prog_off = p->prog_off;
  g.state_off = p->state_off;
  g.rows_off = p->rows_off;
  g.ckpt_off = p->ckpt_off;
  g.bp_off = p->bp_off;
  g.ckpt_bytes = p->ckpt_bytes;
  g.bp_stage = p->bp_stage;
  g.part_bytes = p->part_bytes;
  return g;
}

static int check_plan(const sp_grid_plan* p, int part) {
  if (!p || p->nparts < 1 || p->nparts > kMaxParts || part < 0 || part >= p->nparts || p->part_bytes == 0) {
    set_error(SP_ERR_INVALID, "bad grid plan or partition index %d", part);
    return SP_ERR_INVALID;
  }
  return SP_OK;
}

int sp_grid_plan_make(const sp_instances* in, int32_t nparts, int32_t ctas_per_part, size_t part_ws_bytes,
                      int32_t force_segment, sp_grid_plan* plan, void* ws, size_t ws_bytes, void* stream) {
  int rc = validate(in);
  if (rc) return rc;
  if (in->n != 1 || !plan || nparts < 1 || nparts > kMaxParts) {
    set_error(SP_ERR_INVALID, "sp_grid_plan_make takes exactly one instance and 1..%d partitions", kMaxParts);
    return SP_ERR_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t L = in->total_layers;
  Carve cv{(uint8_t*)ws, ws_bytes};
  InstInfo* info = (InstInfo*)cv.take(sizeof(InstInfo));
  StageShift* shifts = (StageShift*)cv.take(sizeof(StageShift) * L);
  int64_t* rv = (int64_t*)cv.take(sizeof(int64_t) * L);
  int2* reach = (int2*)cv.take(sizeof(int2) * L);
  if (!ws || align_up(cv.used, 256) > ws_bytes) {
    set_required_workspace(align_up(cv.used, 256));
    set_error(SP_ERR_WORKSPACE, "sp_grid_plan_make needs %zu B of scratch", align_up(cv.used, 256));
    return SP_ERR_WORKSPACE;
  }
  prep_kernel<<<1, 128, 0, st>>>(*in, info, shifts, rv, reach, nullptr);
  rc = launch_check("prep_kernel launch");
  InstInfo hinfo;
  uint8_t sac = 0;
  int64_t off0 = 0;
  if (!rc) rc = check_cuda(cudaMemcpyAsync(&hinfo, info, sizeof(hinfo), cudaMemcpyDeviceToHost, st), "copy info");
  if (!rc) rc = check_cuda(cudaMemcpyAsync(&sac, in->source_at_client, 1, cudaMemcpyDeviceToHost, st), "copy sac");
  if (!rc) rc = check_cuda(cudaMemcpyAsync(&off0, in->layer_off, 8, cudaMemcpyDeviceToHost, st), "copy offset");
  int ms = 0;
  if (!rc) rc = read_max_shift(shifts, (int)L, st, &ms);
  if (rc) return rc;
  if (off0 != 0) {
    set_error(SP_ERR_INVALID, "layer_off[0] must be 0");
    return SP_ERR_INVALID;
  }
  const int64_t ncol = hinfo.w_eff + 1;
  if (ncol > kMaxCols) {
    set_error(SP_ERR_UNSUPPORTED, "W_eff = %lld exceeds the supported 2^31 columns", (long long)hinfo.w_eff);
    return SP_ERR_UNSUPPORTED;
  }
  const int resident = grid_resident_rt(hinfo.mode);
  if (resident <= 0) return check_cuda(cudaErrorInvalidConfiguration, "dp_grid_kernel occupancy");
  const int ctas = ctas_per_part > 0 ? std::min(ctas_per_part, resident) : resident;
  GridGeom g;
  bool too_wide = false;
  rc = grid_geometry(hinfo.mode, (int)L, ncol, nparts, ctas, ms, part_ws_bytes / 256 * 256, force_segment, &g,
                     &too_wide);
  if (!rc && too_wide)  // the read-back spans a whole partition: one partition
    rc = grid_geometry(hinfo.mode, (int)L, ncol, 1, ctas, ms, part_ws_bytes / 256 * 256, force_segment, &g,
                       &too_wide);
  if (rc) return rc;
  g.sac = sac ? 1 : 0;
  sp_grid_plan p = {};
  p.mode = g.mode;
  p.n_layers = g.L;
  p.ctas = g.G;
  p.chunks_per_cta = g.NC;
  p.nparts = g.nparts;
  p.seg_stages = g.K;
  p.nseg = g.nseg;
  p.nckpt = g.nckpt;
  p.sac = g.sac;
  p.owner_part = g.owner_part();
  p.ncol = g.ncol;
  p.part_cols = g.Wp;
  p.halo = g.halo;
  p.span = g.span;
  p.row_words = g.row_words;
  p.rec_off = g.rec_off;
  p.prog_off = g.prog_off;
  p.state_off = g.state_off;
  p.rows_off = g.rows_off;
  p.ckpt_off = g.ckpt_off;
  p.bp_off = g.bp_off;
  p.ckpt_bytes = g.ckpt_bytes;
  p.bp_stage = g.bp_stage;
  p.part_bytes = g.part_bytes;
  *plan = p;
  return SP_OK;
}

int sp_grid_part_prepare(const sp_grid_plan* plan, const sp_instances* in, void* part_ws, void* stream) {
  int rc = check_plan(plan, 0);
  if (!rc) rc = validate(in);
  if (rc) return rc;
  if (in->n != 1 || in->total_layers != plan->n_layers || !part_ws) {
    set_error(SP_ERR_INVALID, "sp_grid_part_prepare: the plan's single instance and a workspace");
    return SP_ERR_INVALID;
  }
  const GridGeom g = geom_of(plan);
  uint8_t* pw = (uint8_t*)part_ws;
  cudaStream_t st = (cudaStream_t)stream;
  rc = check_cuda(cudaMemsetAsync(g.state(pw), 0, 128, st), "zero partition state");
  if (rc) return rc;
  prep_kernel<<<1, 128, 0, st>>>(*in, g.info(pw), g.shifts(pw), g.rv(pw), g.reach(pw), nullptr);
  return launch_check("prep_kernel launch");
}

int sp_grid_part_reset(const sp_grid_plan* plan, void* part_ws, void* stream) {
  int rc = check_plan(plan, 0);
  if (rc) return rc;
  const GridGeom g = geom_of(plan);
  return check_cuda(cudaMemsetAsync(g.prog((uint8_t*)part_ws), 0, (size_t)g.G * 4, (cudaStream_t)stream),
                    "zero progress counters");
}

int sp_grid_part_forward(const sp_grid_plan* plan, int32_t part, void* const* part_ws, int32_t seg,
                         int32_t write_ckpt, int32_t keep_bp, void* stream) {
  int rc = check_plan(plan, part);
  if (rc) return rc;
  if (!part_ws || seg < 0 || seg >= plan->nseg) {
    set_error(SP_ERR_INVALID, "sp_grid_part_forward: segment %d of %d", seg, plan->nseg);
    return SP_ERR_INVALID;
  }
  for (int p = 0; p < plan->nparts; ++p)
    if (!part_ws[p]) {
      set_error(SP_ERR_INVALID, "partition %d workspace not mapped", p);
      return SP_ERR_INVALID;
    }
  const GridGeom g = geom_of(plan);
  uint8_t* pw[kMaxParts] = {};
  for (int p = 0; p < g.nparts; ++p) pw[p] = (uint8_t*)part_ws[p];
  const int k0 = g.seg_begin(seg), cnt = g.seg_begin(seg + 1) - k0;
  GridArgs a = grid_args(g, pw, k0, cnt, seg, write_ckpt ? seg + 1 : 0, keep_bp != 0, 1);
  a.part_base = part;
  a.launch_parts = 1;
  grid_set_records(a, g, pw[part], true);
  return launch_grid(g.mode, a, (cudaStream_t)stream);
}

int sp_grid_part_end(const sp_grid_plan* plan, void* owner_ws, int8_t must_end_at, int64_t* state, void* stream) {
  int rc = check_plan(plan, plan ? plan->owner_part : 0);
  if (rc) return rc;
  if (!owner_ws || !state) {
    set_error(SP_ERR_INVALID, "sp_grid_part_end: null workspace or state");
    return SP_ERR_INVALID;
  }
  const GridGeom g = geom_of(plan);
  uint8_t* pw = (uint8_t*)owner_ws;
  grid_end_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(g.info(pw), (int64_t)plan->owner_part * g.Wp, g.Wp, g.L,
                                                      must_end_at, nullptr, g.ckpt(pw, g.nseg), state);
  return launch_check("grid_end_kernel launch");
}

int sp_grid_part_backtrack(const sp_grid_plan* plan, int32_t part, void* part_ws, int32_t seg, int64_t* state,
                           uint8_t* pi, void* stream) {
  int rc = check_plan(plan, part);
  if (rc) return rc;
  if (!part_ws || !state || !pi || seg < 0 || seg >= plan->nseg) {
    set_error(SP_ERR_INVALID, "sp_grid_part_backtrack: bad arguments");
    return SP_ERR_INVALID;
  }
  const GridGeom g = geom_of(plan);
  uint8_t* pw = (uint8_t*)part_ws;
  const int k0 = g.seg_begin(seg), cnt = g.seg_begin(seg + 1) - k0;
  grid_backtrack_part_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(g.shifts(pw), g.bp(pw), g.row_words, g.mode, k0,
                                                                 cnt, (int64_t)part * g.Wp, state, pi);
  return launch_check("grid_backtrack_part_kernel launch");
}

// ---- CUDA IPC of partition workspaces (one process per device) --------------

typedef int (*AddrRangeFn)(unsigned long long*, size_t*, unsigned long long);

int sp_ipc_export(const void* dptr, void* handle, size_t* offset) {
  if (!dptr || !handle || !offset) {
    set_error(SP_ERR_INVALID, "sp_ipc_export: null argument");
    return SP_ERR_INVALID;
  }
  // the handle names the whole allocation: find its base through the driver
  // entry point (no libcuda link dependency)
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  int rc = check_cuda(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q),
                      "cudaGetDriverEntryPoint(cuMemGetAddressRange)");
  if (rc) return rc;
  if (!fn || q != cudaDriverEntryPointSuccess) {
    set_error(SP_ERR_CUDA, "cuMemGetAddressRange unavailable");
    return SP_ERR_CUDA;
  }
  unsigned long long base = 0;
  size_t size = 0;
  if (((AddrRangeFn)fn)(&base, &size, (unsigned long long)(uintptr_t)dptr) != 0) {
    set_error(SP_ERR_CUDA, "cuMemGetAddressRange failed");
    return SP_ERR_CUDA;
  }
  cudaIpcMemHandle_t h;
  rc = check_cuda(cudaIpcGetMemHandle(&h, (void*)(uintptr_t)base), "cudaIpcGetMemHandle");
  if (rc) return rc;
  memcpy(handle, &h, sizeof(h));
  *offset = (size_t)((uintptr_t)dptr - (uintptr_t)base);
  return SP_OK;
}

int sp_ipc_import(const void* handle, size_t offset, void** dptr, void** base) {
  if (!handle || !dptr || !base) {
    set_error(SP_ERR_INVALID, "sp_ipc_import: null argument");
    return SP_ERR_INVALID;
  }
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* p = nullptr;
  int rc = check_cuda(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  if (rc) return rc;
  *base = p;
  *dptr = (uint8_t*)p + offset;
  return SP_OK;
}

int sp_ipc_close(void* base) { return check_cuda(cudaIpcCloseMemHandle(base), "cudaIpcCloseMemHandle"); }

int sp_build_dp_tables(const sp_instances* in, int64_t w_eff, double* client_table,
                       double* server_table, void* ws, size_t ws_bytes, void* stream) {
  int rc = validate(in);
  if (rc) return rc;
  if (in->n != 1 || !client_table || !server_table) {
    set_error(SP_ERR_INVALID, "sp_build_dp_tables takes exactly one instance and two tables");
    return SP_ERR_INVALID;
  }
  if (w_eff < 0) {
    set_error(SP_ERR_INVALID, "negative w_eff");
    return SP_ERR_INVALID;
  }
  return run_dp(in, nullptr, client_table, server_table, ws, ws_bytes, (cudaStream_t)stream, nullptr, nullptr,
                nullptr, nullptr, nullptr, w_eff);
}


int sp_evaluate_policy(const sp_instances* in, const uint8_t* pi, sp_policies* out, void* ws,
                       size_t ws_bytes, void* stream) {
  int rc = validate(in);
  if (rc) return rc;
  rc = validate_out(out);
  if (rc) return rc;
  if (in->n == 0) return SP_OK;
  if (!pi) {
    set_error(SP_ERR_INVALID, "null pi");
    return SP_ERR_INVALID;
  }
  const size_t need = sizeof(int32_t) * (size_t)in->total_layers;
  if (!ws || ws_bytes < need) {
    set_required_workspace(need);
    set_error(SP_ERR_WORKSPACE, "sp_evaluate_policy needs %zu B of scratch", need);
    return SP_ERR_WORKSPACE;
  }
  evaluate_kernel<<<(unsigned)((in->n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(*in, pi, *out,
                                                                                     (int32_t*)ws);
  return launch_check("evaluate_kernel launch");
}

int sp_plan_prefix(const sp_instances* in, int32_t which, sp_policies* out, void* stream) {
  int rc = validate(in);
  if (rc) return rc;
  rc = validate_out(out);
  if (rc) return rc;
  if (which < SP_GREEDY || which > SP_ALL_CLIENT) {
    set_error(SP_ERR_INVALID, "unknown prefix planner %d", which);
    return SP_ERR_INVALID;
  }
  if (in->n == 0) return SP_OK;
  const int64_t threads = in->n * 32;
  prefix_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, (cudaStream_t)stream>>>(*in, which, *out);
  return launch_check("prefix_kernel launch");
}

int sp_plan_exhaustive(const sp_instances* in, sp_policies* out, void* stream) {
  int rc = validate(in);
  if (rc) return rc;
  rc = validate_out(out);
  if (rc) return rc;
  if (in->n == 0) return SP_OK;
  // L <= 24 (planner.py:21 ORACLE_MAX_LAYERS): the kernel enumerates 2^L masks
  // in 32-bit words and keeps a 32-entry index list
  std::vector<int64_t> hoff(in->n + 1);
  rc = check_cuda(cudaMemcpyAsync(hoff.data(), in->layer_off, sizeof(int64_t) * (in->n + 1),
                                  cudaMemcpyDeviceToHost, (cudaStream_t)stream),
                  "copy layer offsets");
  if (!rc) rc = check_cuda(cudaStreamSynchronize((cudaStream_t)stream), "sync");
  if (rc) return rc;
  for (int64_t k = 0; k < in->n; ++k) {
    const int64_t L = hoff[k + 1] - hoff[k];
    if (L < 0 || L > 24) {
      set_error(SP_ERR_UNSUPPORTED, "oracle limited to 24 layers, got %lld (instance %lld)", (long long)L,
                (long long)k);
      return SP_ERR_UNSUPPORTED;
    }
  }
  exhaustive_kernel<<<(unsigned)in->n, 256, 0, (cudaStream_t)stream>>>(*in, *out);
  return launch_check("exhaustive_kernel launch");
}

int sp_latency_eq1(const sp_instances* in, const double* client_s, const double* server_s,
                   const double* up_s, const double* down_s, const uint8_t* pi, double* latency_s,
                   void* stream) {
  int rc = validate(in);
  if (rc) return rc;
  if (in->n == 0) return SP_OK;
  if (!client_s || !server_s || !up_s || !down_s || !pi || !latency_s) {
    set_error(SP_ERR_INVALID, "null array in sp_latency_eq1");
    return SP_ERR_INVALID;
  }
  eq1_kernel<<<(unsigned)((in->n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      *in, client_s, server_s, up_s, down_s, pi, latency_s);
  return launch_check("eq1_kernel launch");
}

}  // extern "C"
