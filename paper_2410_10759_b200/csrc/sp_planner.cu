// Planner kernels of the B200 placement engine (reference: planner.py).
//
//   dp_core.cuh        prep_kernel (W_eff, value domain, clamped stage shifts,
//                      reachable frontiers), the per-cell update, and
//                      dp_stage_kernel: K2 with rows in one CTA's SMEM
//                      (planner.py:128-143), 2-bit packed back-pointers
//   dp_stream.cuh      K2 for wide rows: dp_stream_kernel (L2 rows, bulk-copy
//                      windows), dp_own_kernel (experiment)
//   dp_grid.cuh        K2 for one huge instance (cfg5): dp_grid_kernel,
//                      dp_grid_inplace_kernel, checkpoint/backtrack kernels
//   dp_cluster_coop.cuh  forced-only K2 variants (parity coverage)
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
#include <type_traits>
#include <vector>

#include "sp_internal.cuh"

namespace sp {
namespace {

constexpr int kStageTile = 128;          // stage records staged in SMEM at a time
constexpr int kCellsPerThread = 4;       // E: columns per thread per chunk
constexpr int kMaxThreads = 1024;
constexpr int kStageThreads = 512;     // single-CTA DP kernels: 2 CTAs per SM
constexpr size_t kSmemCap = 227 * 1024;  // sm_100a max dynamic SMEM per CTA
constexpr int64_t kMaxCols = (int64_t(1) << 31) - 64;

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

#include "dp_core.cuh"
#include "dp_cluster_coop.cuh"
#include "dp_stream.cuh"
#include "dp_grid.cuh"

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
// exhaustive planner (plan_oracle): one CTA per instance, masks strided

__global__ void exhaustive_kernel(sp_instances in, sp_policies out) {
  const int64_t inst = blockIdx.x;
  const int64_t lo = in.layer_off[inst];
  const int L = (int)(in.layer_off[inst + 1] - lo);
  const bool sac = in.source_at_client[inst] != 0;
  const int64_t budget = in.budget[inst];
  __shared__ double s_val[32];
  __shared__ uint32_t s_mask[32];
  __shared__ int s_found[32];
  double best_v = -INFINITY;
  uint32_t best_m = 0xffffffffu;
  int found = 0;
  const uint32_t nmask = 1u << L;
  for (uint32_t mask = threadIdx.x; mask < nmask; mask += blockDim.x) {
    int64_t lat = 0;
    double v = 0.0;
    int prev = sac ? 1 : 0;
    for (int k = 0; k < L; ++k) {
      const int x = (mask >> (L - 1 - k)) & 1;  // layer 1 is the MSB
      if (x) {
        lat += in.client_units[lo + k] + (prev ? 0 : in.down_units[lo + k]);
        v = dadd(v, in.r[lo + k]);
      } else {
        lat += in.server_units[lo + k] + (prev ? in.up_units[lo + k] : 0);
      }
      prev = x;
    }
    if (lat <= budget && (!found || v > best_v || (v == best_v && mask < best_m))) {
      best_v = v;
      best_m = mask;
      found = 1;
    }
  }
  // warp + block arg-reduction: larger value, then smaller mask
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, best_v, o);
    const uint32_t om = __shfl_xor_sync(0xffffffffu, best_m, o);
    const int of = __shfl_xor_sync(0xffffffffu, found, o);
    if (of && (!found || ov > best_v || (ov == best_v && om < best_m))) {
      best_v = ov;
      best_m = om;
      found = 1;
    }
  }
  if (lane == 0) {
    s_val[wid] = best_v;
    s_mask[wid] = best_m;
    s_found[wid] = found;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nw = blockDim.x / 32;
    for (int w = 1; w < nw; ++w) {
      if (s_found[w] && (!found || s_val[w] > best_v || (s_val[w] == best_v && s_mask[w] < best_m))) {
        best_v = s_val[w];
        best_m = s_mask[w];
        found = 1;
      }
    }
    uint8_t* pi = out.pi + lo;
    for (int k = 0; k < L; ++k) pi[k] = found ? (uint8_t)((best_m >> (L - 1 - k)) & 1) : 0;
    int32_t idx[32];  // L <= 24 (planner.py:21 ORACLE_MAX_LAYERS)
    finish_policy(in, inst, lo, L, idx, out, !found, false);
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

enum DpVariant { DPV_SMEM = 0, DPV_CLUSTER = 1, DPV_GLOBAL = 2, DPV_COOP = 3, DPV_STREAM = 4, DPV_OWN = 6 };

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
// row buffers of the streaming kernel: 2 (full-barrier semantics, default:
// 2/3 of the L2 footprint lets G shrink to 5 at W = 1e5, measured 4.5e11 vs
// 4.4e11 cells/s with 3) or 3 (one stage of slack); SPLITPLAN_STREAM_BUFS
int stream_bufs() {
  static int b = 0;
  if (!b) b = env_int("SPLITPLAN_STREAM_BUFS", 2) == 3 ? 3 : 2;
  return b;
}
size_t stream_row_bytes(int mode, const StreamGeom& g) {
  return 2 * (size_t)stream_bufs() * (size_t)stream_span(mode, g) * value_bytes(mode);
}

// instances per cluster of the streaming kernel (1 or 2; SPLITPLAN_STREAM_PAIR,
// 256 x 4 only).  Pairs were measured slower on B200 (3.4-4.1e11 vs 4.4e11
// cells/s at W = 1e5: the doubled L2 footprint costs more than the hidden
// stage latency saves).
int stream_pair() {
  static int p = 0;
  if (!p) p = env_int("SPLITPLAN_STREAM_PAIR", 1) == 2 ? 2 : 1;
  return p;
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
// every co-resident instance (stream_pair() per cluster) fit the L2 budget;
// among those, the G minimising G * (NC * CH + sync) -- the CTA-time of one
// stage in columns, padding waste included, plus the stage-synchronisation
// latency per CTA (about 4096 columns for single instances, measured on
// B200; paired instances hide most of it behind the partner's stage).
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
  const int pair = cfg == 0 ? stream_pair() : 1;
  const int64_t sync = pair == 2 ? 0 : 4096;
  auto cost_of = [&](const StreamGeom& t) { return (int64_t)t.G * ((int64_t)t.NC * ch + sync); };
  if (force >= 1 && force <= 16) {
    const StreamGeom t = geom(force);
    *cost = cost_of(t);
    return t;
  }
  int gmin = 16;
  for (int G = 1; G <= 16; ++G)
    if ((size_t)(resident / G) * pair * stream_row_bytes(mode, geom(G)) <= l2_row_budget()) {
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
  const int sel = (stream_pair() == 2 ? 1 : 0) + (stream_bufs() == 2 ? 2 : 0);
  switch (sel) {
    case 0: return launch_stream_t<MODE, 256, 4, NS, 1, 3>(a, n_items, geo, st);
    case 1: return launch_stream_t<MODE, 256, 4, NS, 2, 3>(a, n_items, geo, st);
    case 2: return launch_stream_t<MODE, 256, 4, NS, 1, 2>(a, n_items, geo, st);
    default: return launch_stream_t<MODE, 256, 4, NS, 2, 2>(a, n_items, geo, st);
  }
}

// ---- own-block kernel (int32 rows in the cluster's shared memory) ----------

struct OwnCfg {
  int T, E, NSW;
};
constexpr OwnCfg kOwnCfgs[] = {{512, 4, 8}, {256, 8, 8}, {256, 4, 8}};
int own_cfg_index() {
  const int c = env_int("SPLITPLAN_OWN_CFG", 0);
  return c < 0 || c > 2 ? 0 : c;
}
// CTAs per SM the own-block geometry is sized for (SPLITPLAN_OWN_OCC 1 or 2)
size_t own_smem_budget() {
  return env_int("SPLITPLAN_OWN_OCC", 1) == 2 ? (size_t)113 * 1024 : kSmemCap;
}
// global row buffers (3: one stage of slack for the wavefront; SPLITPLAN_OWN_BUFS 2..4)
int own_bufs() { return std::min(4, std::max(2, env_int("SPLITPLAN_OWN_BUFS", 3))); }
int64_t own_ch() { return (int64_t)kOwnCfgs[own_cfg_index()].T * kOwnCfgs[own_cfg_index()].E; }
size_t own_smem(int mode, int NC) {
  const size_t vb = value_bytes(mode);
  const int64_t ch = own_ch();
  return 256 + (size_t)(2 * (ch + NC * ch) + kOwnCfgs[own_cfg_index()].NSW * (ch + 16 / (int64_t)vb)) * vb;
}
// cluster geometry: the fewest CTAs whose blocks fit shared memory (G = 0: not possible)
StreamGeom own_geom(int mode, int64_t ncol) {
  StreamGeom g{0, 0, 0, 0, 0};
  if (mode != VM_INT32) return g;
  const int64_t nchunks = (ncol + own_ch() - 1) / own_ch();
  int ncmax = 0;
  while (own_smem(mode, ncmax + 1) <= own_smem_budget()) ++ncmax;
  if (ncmax < 1) return g;
  int G = (int)((nchunks + ncmax - 1) / ncmax);
  const int force = env_int("SPLITPLAN_DP_CLUSTER", 0);
  if (force >= 1 && force <= 16) G = std::max(G, force);
  if (G > 16) return g;
  const int NC = (int)((nchunks + G - 1) / G);
  g.G = (int)((nchunks + NC - 1) / NC);
  g.NC = NC;
  return g;
}
int64_t own_span(int mode, const StreamGeom& g) {
  const int64_t line = 128 / (int64_t)value_bytes(mode);
  return (own_ch() + line) + (int64_t)g.G * g.NC * own_ch() + line;
}
size_t own_row_bytes(int mode, const StreamGeom& g) {
  return 2 * (size_t)own_bufs() * (size_t)own_span(mode, g) * value_bytes(mode);
}

template <int MODE, int T, int E, int NSW, int NBUF>
int launch_own_t(const DpArgs& a, int64_t n_items, StreamGeom sg, size_t smem, cudaStream_t st) {
  auto kern = dp_own_kernel<MODE, T, E, NSW, NBUF>;
  int rc = check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                      "cudaFuncSetAttribute(dp_own_kernel)");
  if (rc) return rc;
  if (sg.G > 8) {
    rc = check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
                    "cudaFuncSetAttribute(non-portable cluster)");
    if (rc) return rc;
  }
  OwnGeom geo{sg.G, sg.NC, (int)n_items, 0};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(n_items * sg.G), 1, 1);
  cfg.blockDim = dim3((unsigned)(T + 64), 1, 1);  // + producer and publisher warps
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)sg.G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  rc = check_cuda(cudaLaunchKernelEx(&cfg, kern, a, geo), "dp_own_kernel launch");
  if (rc) return rc;
  return launch_check("dp_own_kernel launch");
}
int launch_own(int mode, const DpArgs& a, int64_t n_items, StreamGeom sg, size_t smem, cudaStream_t st) {
  if (mode != VM_INT32) return check_cuda(cudaErrorInvalidValue, "dp_own_kernel: int32 domain only");
  const int sel = own_cfg_index() * 3 + (own_bufs() - 2);
  switch (sel) {
    case 6: return launch_own_t<VM_INT32, 256, 4, 8, 2>(a, n_items, sg, smem, st);
    case 7: return launch_own_t<VM_INT32, 256, 4, 8, 3>(a, n_items, sg, smem, st);
    case 8: return launch_own_t<VM_INT32, 256, 4, 8, 4>(a, n_items, sg, smem, st);
    case 0: return launch_own_t<VM_INT32, 512, 4, 8, 2>(a, n_items, sg, smem, st);
    case 1: return launch_own_t<VM_INT32, 512, 4, 8, 3>(a, n_items, sg, smem, st);
    case 2: return launch_own_t<VM_INT32, 512, 4, 8, 4>(a, n_items, sg, smem, st);
    case 3: return launch_own_t<VM_INT32, 256, 8, 8, 2>(a, n_items, sg, smem, st);
    case 4: return launch_own_t<VM_INT32, 256, 8, 8, 3>(a, n_items, sg, smem, st);
    case 5: return launch_own_t<VM_INT32, 256, 8, 8, 4>(a, n_items, sg, smem, st);
    default: return launch_own_t<VM_INT32, 512, 4, 8, 3>(a, n_items, sg, smem, st);
  }
}

// ---- cluster (DSMEM rows) and cooperative (L2 rows, LDG) kernels ------------

template <int MODE>
int launch_cluster(const DpArgs& a, int64_t n_items, int threads, size_t smem, ClusterGeom geo,
                   cudaStream_t st) {
  auto kern = dp_cluster_kernel<MODE>;
  // the kernel also has a little static SMEM, so ask for exactly what it uses
  int rc = check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem),
                      "cudaFuncSetAttribute(dp_cluster_kernel)");
  if (rc) return rc;
  if (geo.G > 8) {
    rc = check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
                    "cudaFuncSetAttribute(non-portable cluster)");
    if (rc) return rc;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(n_items * geo.G), 1, 1);
  cfg.blockDim = dim3((unsigned)threads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)geo.G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  rc = check_cuda(cudaLaunchKernelEx(&cfg, kern, a, geo), "dp_cluster_kernel launch");
  if (rc) return rc;
  return launch_check("dp_cluster_kernel launch");
}

template <int MODE>
int launch_coop(const DpArgs& a, int64_t n_items, int threads, size_t smem, ClusterGeom geo,
                cudaStream_t st) {
  auto kern = dp_coop_kernel<MODE, kCellsPerThread>;
  int rc = SP_OK;
  if (geo.G > 8) {
    rc = check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
                    "cudaFuncSetAttribute(non-portable cluster)");
    if (rc) return rc;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(n_items * geo.G), 1, 1);
  cfg.blockDim = dim3((unsigned)threads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)geo.G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  rc = check_cuda(cudaLaunchKernelEx(&cfg, kern, a, geo), "dp_coop_kernel launch");
  if (rc) return rc;
  return launch_check("dp_coop_kernel launch");
}

// cooperative geometry: enough CTAs per instance that the double-buffered
// rows of every co-resident instance fit comfortably in L2
ClusterGeom coop_geom(int mode, int64_t ncol) {
  const size_t vb = value_bytes(mode);
  const size_t l2_budget = (size_t)48 << 20;
  const int resident_ctas = 148 * 2;
  int G = 2;
  for (; G < 16; G *= 2) {
    const int64_t B = ((ncol + G - 1) / G + 31) / 32 * 32;
    const int64_t t = std::min<int64_t>(kStageThreads, std::max<int64_t>(32, ((B + 3) / 4 + 31) / 32 * 32));
    const size_t per_inst = 4 * (size_t)(kCellsPerThread * t + ncol) * vb;
    if ((size_t)(resident_ctas / G) * per_inst <= l2_budget) break;
  }
  ClusterGeom geo;
  geo.G = G;
  geo.B = (int)(((ncol + G - 1) / G + 31) / 32 * 32);
  geo.magic = 0;
  return geo;
}

int coop_threads(const ClusterGeom& geo) {
  return (int)std::min<int64_t>(kStageThreads,
                                std::max<int64_t>(32, ((geo.B + 3) / 4 + 31) / 32 * 32));
}

size_t coop_row_bytes(int mode, int64_t ncol, const ClusterGeom& geo) {
  return 4 * (size_t)(kCellsPerThread * coop_threads(geo) + ncol) * value_bytes(mode);
}

// cluster geometry for one instance, or G == 0 if the rows do not fit on chip
ClusterGeom cluster_geom(int mode, int64_t ncol) {
  ClusterGeom geo{0, 0, 0};
  const size_t vb = value_bytes(mode);
  const size_t room = kSmemCap - stage_bytes_mode(mode) - 1024;  // 1 KB for static SMEM
  const size_t per_col = 4 * vb;  // 2 buffers x (C, S)
  int G = (int)((ncol * per_col + room - 1) / room);
  G = std::max(G, 2);
  if (G > 16) return geo;
  // B: a multiple of 32 so every warp's columns form one packed back-pointer group
  const int64_t B = ((ncol + G - 1) / G + 31) / 32 * 32;
  if ((size_t)B * per_col > room) return geo;
  const uint64_t magic = ((uint64_t)1 << 32) / (uint64_t)B + 1;
  // umulhi(x, magic) == x / B for all x < N whenever N * B < 2^32
  // (magic * B - 2^32 <= B, so the error term x * that / 2^32 stays below 1/B)
  if ((uint64_t)G * (uint64_t)B * (uint64_t)B >= ((uint64_t)1 << 32)) return geo;
  geo.G = G;
  geo.B = (int)B;
  geo.magic = (uint32_t)magic;
  return geo;
}

int forced_variant() {
  const char* v = getenv("SPLITPLAN_DP_VARIANT");
  if (!v) return -1;
  if (!strcmp(v, "smem")) return DPV_SMEM;
  if (!strcmp(v, "cluster")) return DPV_CLUSTER;
  if (!strcmp(v, "global")) return DPV_GLOBAL;
  if (!strcmp(v, "coop")) return DPV_COOP;
  if (!strcmp(v, "stream")) return DPV_STREAM;
  if (!strcmp(v, "grid")) return 5;  // DPV_GRID
  if (!strcmp(v, "own")) return DPV_OWN;
  return -1;
}

// Launch plan of one instance: kernel variant, its configuration, and the
// workspace / shared memory it needs.
struct DpPlan {
  int variant = DPV_SMEM;
  int cfg = 0;                  // single-CTA T x E configuration
  int threads = 0;
  ClusterGeom cgeo{0, 0, 0};    // cluster / coop
  StreamGeom sgeo{0, 0, 0, 0};  // stream
  size_t bp = 0, rows = 0, smem = 0;
  int64_t bp_row_words = 0;
  // launches sharing a key go out together
  bool same_launch(const DpPlan& o) const {
    return variant == o.variant && cfg == o.cfg && threads == o.threads && cgeo.G == o.cgeo.G &&
           cgeo.B == o.cgeo.B && sgeo.G == o.sgeo.G && sgeo.NC == o.sgeo.NC && sgeo.cfg == o.sgeo.cfg;
  }
};

DpPlan plan_instance(int mode, int64_t L, int64_t ncol, int force, bool tables) {
  DpPlan p;
  const size_t vb = value_bytes(mode);
  p.cfg = single_cfg_for(ncol, (force == DPV_GLOBAL || tables) ? VM_F64 : mode);
  const size_t single_rows = single_row_bytes(mode, ncol, p.cfg);
  const bool fits_cta = single_rows + stage_bytes_mode(mode) <= kSmemCap;
  if (force == DPV_GLOBAL || (tables && force < 0)) p.variant = DPV_GLOBAL;
  else if (force == DPV_SMEM && fits_cta) p.variant = DPV_SMEM;
  else if (force == DPV_CLUSTER && cluster_geom(mode, ncol).G) p.variant = DPV_CLUSTER;
  else if (force == DPV_COOP) p.variant = DPV_COOP;
  else if (force == DPV_STREAM) p.variant = DPV_STREAM;
  else if (force == DPV_OWN && own_geom(mode, ncol).G) p.variant = DPV_OWN;
  else if (fits_cta && force != DPV_CLUSTER) p.variant = DPV_SMEM;
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
    case DPV_OWN:
      p.sgeo = own_geom(mode, ncol);
      p.threads = kOwnCfgs[own_cfg_index()].T;
      p.bp_row_words = bp_row_words_for(mode, (int64_t)p.sgeo.G * p.sgeo.NC * own_ch());
      p.rows = align_up(own_row_bytes(mode, p.sgeo), 256);
      p.smem = own_smem(mode, p.sgeo.NC);
      break;
    case DPV_COOP:
      p.cgeo = coop_geom(mode, ncol);
      p.threads = coop_threads(p.cgeo);
      p.bp_row_words = bp_row_words_for(mode, ncol);
      p.rows = align_up(coop_row_bytes(mode, ncol, p.cgeo), 256);
      p.smem = stage_bytes_mode(mode);
      break;
    case DPV_CLUSTER:
      p.cgeo = cluster_geom(mode, ncol);
      p.threads = (int)std::min<int64_t>(kMaxThreads,
                                         std::max<int64_t>(64, ((p.cgeo.B + 3) / 4 + 31) / 32 * 32));
      p.bp_row_words = bp_row_words_for(mode, ncol);
      p.smem = stage_bytes_mode(mode) + 4 * vb * (size_t)p.cgeo.B;
      break;
  }
  p.bp = align_up((size_t)L * (size_t)p.bp_row_words * 4, 256);
  return p;
}

int launch_plan(int mode, const DpPlan& p, const DpArgs& a, int64_t n_items, cudaStream_t st) {
  if (n_items == 0) return SP_OK;
  switch (p.variant) {
    case DPV_OWN:
      return launch_own(mode, a, n_items, p.sgeo, p.smem, st);
    case DPV_STREAM:
      switch (mode) {
        case VM_INT32: return launch_stream<VM_INT32>(a, n_items, p.sgeo, st);
        case VM_F64: return launch_stream<VM_F64>(a, n_items, p.sgeo, st);
        default: return launch_stream<VM_F64_NAN>(a, n_items, p.sgeo, st);
      }
    case DPV_COOP:
      switch (mode) {
        case VM_INT32: return launch_coop<VM_INT32>(a, n_items, p.threads, p.smem, p.cgeo, st);
        case VM_F64: return launch_coop<VM_F64>(a, n_items, p.threads, p.smem, p.cgeo, st);
        default: return launch_coop<VM_F64_NAN>(a, n_items, p.threads, p.smem, p.cgeo, st);
      }
    case DPV_CLUSTER:
      switch (mode) {
        case VM_INT32: return launch_cluster<VM_INT32>(a, n_items, p.threads, p.smem, p.cgeo, st);
        case VM_F64: return launch_cluster<VM_F64>(a, n_items, p.threads, p.smem, p.cgeo, st);
        default: return launch_cluster<VM_F64_NAN>(a, n_items, p.threads, p.smem, p.cgeo, st);
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

template <int MODE>
int launch_grid_inplace_t(const GridInplaceArgs& g, cudaStream_t st) {
  auto kern = dp_grid_inplace_kernel<MODE, kGridT, grid_e<MODE>(), grid_slots<MODE>()>;
  int rc0 = check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)grid_smem(MODE)),
                       "cudaFuncSetAttribute(dp_grid_inplace_kernel)");
  if (rc0) return rc0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)g.G, 1, 1);
  cfg.blockDim = dim3((unsigned)(kGridT + 32), 1, 1);
  cfg.dynamicSmemBytes = grid_smem(MODE);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // every CTA co-resident: the waits are safe
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int rc = check_cuda(cudaLaunchKernelEx(&cfg, kern, g), "dp_grid_inplace_kernel launch");
  if (rc) return rc;
  return launch_check("dp_grid_inplace_kernel launch");
}
int launch_grid_inplace(int mode, const GridInplaceArgs& g, cudaStream_t st) {
  switch (mode) {
    case VM_INT32: return launch_grid_inplace_t<VM_INT32>(g, st);
    case VM_F64: return launch_grid_inplace_t<VM_F64>(g, st);
    default: return launch_grid_inplace_t<VM_F64_NAN>(g, st);
  }
}

int launch_grid(int mode, const GridArgs& g, cudaStream_t st) {
  switch (mode) {
    case VM_INT32: return launch_grid_t<VM_INT32>(g, st);
    case VM_F64: return launch_grid_t<VM_F64>(g, st);
    default: return launch_grid_t<VM_F64_NAN>(g, st);
  }
}

__global__ void zero_progs_kernel(GridArgs g) {
  for (int p = 0; p < g.nparts; ++p)
    for (int x = threadIdx.x; x < g.G; x += blockDim.x) g.progs[p][x] = 0u;
}

// Devices of the calling thread's sp_plan_dp_devices call (empty otherwise).
thread_local std::vector<int> tl_grid_devices;

// Partitions on other devices (SPLITPLAN_GRID_DEVICES > 1): their row buffers,
// progress counters and stage-record copies live in that device's memory;
// every device reaches the others' (and the caller's workspace) through peer
// access.  Released when the solve returns.
struct PeerParts {
  int cur = 0;
  int dev[kMaxParts] = {};
  cudaStream_t stream[kMaxParts] = {};
  cudaEvent_t done[kMaxParts] = {};
  std::vector<std::pair<int, void*>> allocs;
  cudaEvent_t start = nullptr;
  ~PeerParts() {
    for (int p = 0; p < kMaxParts; ++p) {
      if (!stream[p]) continue;
      cudaSetDevice(dev[p]);
      cudaStreamSynchronize(stream[p]);
      cudaStreamDestroy(stream[p]);
      if (done[p]) cudaEventDestroy(done[p]);
    }
    for (auto& a : allocs) {
      cudaSetDevice(a.first);
      cudaFree(a.second);
    }
    cudaSetDevice(cur);
    if (start) cudaEventDestroy(start);
  }
  void* alloc(int d, size_t bytes) {
    void* ptr = nullptr;
    cudaSetDevice(d);
    if (cudaMalloc(&ptr, bytes) != cudaSuccess) ptr = nullptr;
    else allocs.push_back({d, ptr});
    cudaSetDevice(cur);
    return ptr;
  }
};

// Workspace of the whole-GPU path for one instance on one device (single
// partition): the smallest that runs it (checkpoint / recompute with
// ~sqrt(L) segments) and the one that keeps every back-pointer stage.
void grid_workspace_bytes(int mode, int64_t L, int64_t ncol, size_t* min_bytes, size_t* full_bytes) {
  const size_t vb = value_bytes(mode);
  const int resident = mode == VM_INT32 ? grid_resident<VM_INT32>()
                       : mode == VM_F64 ? grid_resident<VM_F64>()
                                        : grid_resident<VM_F64_NAN>();
  const int64_t nchunks = (ncol + grid_ch(mode) - 1) / grid_ch(mode);
  int G = (int)std::max<int64_t>(1, std::min<int64_t>(std::max(resident, 1), nchunks));
  const int NC = (int)((nchunks + G - 1) / G);
  G = (int)((nchunks + NC - 1) / NC);
  const int64_t B = (int64_t)NC * grid_ch(mode), line = 128 / (int64_t)vb;
  const int64_t span = (grid_ch(mode) + line) + G * B + line;
  const size_t bp_stage = (size_t)bp_row_words_for(mode, G * B) * 4;
  const size_t ckpt = align_up(2 * (size_t)ncol * vb, 256);
  const size_t fixed = align_up((size_t)G * 4, 256) + 256 + align_up(2 * kRowBufs * (size_t)span * vb, 256);
  auto need = [&](int64_t k) {
    const size_t nseg = (size_t)((L + k - 1) / k);
    return fixed + (k == L ? 2 : nseg + 1) * ckpt + align_up((size_t)k * bp_stage, 256);
  };
  int64_t K = std::max<int64_t>(1, (int64_t)std::sqrt((double)L * (double)ckpt / (double)bp_stage));
  K = std::min(K, L);
  *min_bytes = need(K);
  *full_bytes = need(L);
}

// Solve one instance over the whole GPU.  With the full back-pointer table in
// memory: one forward launch and one backtrack.  Otherwise checkpoint /
// recompute: a forward pass that keeps a row every K stages, then, segment by
// segment from the end, a recompute of the segment's back-pointers from its
// checkpoint and a backtrack through it (2x the DP work, sqrt(L) memory).
int run_grid_instance_parts(const sp_instances* in, sp_policies* out, InstInfo* info,
                            const StageShift* shifts, const int64_t* rv, const int2* reach, int32_t* idx,
                            int64_t inst, int64_t lo, int L, int64_t ncol, int mode, uint8_t* dyn, size_t avail,
                            cudaStream_t st, int force_parts);

int run_grid_instance(const sp_instances* in, sp_policies* out, InstInfo* info, const StageShift* shifts,
                      const int64_t* rv, const int2* reach, int32_t* idx, int64_t inst, int64_t lo, int L,
                      int64_t ncol, int mode, uint8_t* dyn, size_t avail, cudaStream_t st) {
  return run_grid_instance_parts(in, out, info, shifts, rv, reach, idx, inst, lo, L, ncol, mode, dyn, avail, st,
                                 0);
}

int run_grid_instance_parts(const sp_instances* in, sp_policies* out, InstInfo* info,
                            const StageShift* shifts, const int64_t* rv, const int2* reach, int32_t* idx,
                            int64_t inst, int64_t lo, int L, int64_t ncol, int mode, uint8_t* dyn, size_t avail,
                            cudaStream_t st, int force_parts) {
  const size_t vb = value_bytes(mode);
  const int resident = mode == VM_INT32 ? grid_resident<VM_INT32>()
                       : mode == VM_F64 ? grid_resident<VM_F64>()
                                        : grid_resident<VM_F64_NAN>();
  if (resident <= 0) return check_cuda(cudaErrorInvalidConfiguration, "dp_grid_kernel occupancy");
  const int64_t nchunks = (ncol + grid_ch(mode) - 1) / grid_ch(mode);
  // partitions of the capacity axis (one per device in a multi-GPU run;
  // SPLITPLAN_GRID_PARTS > 1 emulates them on this device)
  // SPLITPLAN_GRID_DEVICES > 1 places partition p on device (current + p),
  // one launch per device; SPLITPLAN_GRID_SEPARATE=1 runs emulated partitions
  // as separate concurrent launches on this device (the multi-device protocol
  // with every partition here).
  int ndev_avail = 1;
  if (cudaGetDeviceCount(&ndev_avail) != cudaSuccess) {
    cudaGetLastError();
    ndev_avail = 1;
  }
  // partition -> device: sp_plan_dp_devices' list, else SPLITPLAN_GRID_DEVICES
  // consecutive devices from the current one
  int cur_dev = 0;
  cudaGetDevice(&cur_dev);
  std::vector<int> devlist = tl_grid_devices;
  if (devlist.empty()) {
    const int n = std::max(1, std::min(std::min(kMaxParts, ndev_avail), env_int("SPLITPLAN_GRID_DEVICES", 1)));
    for (int p = 0; p < n; ++p) devlist.push_back((cur_dev + p) % ndev_avail);
  }
  if ((int)devlist.size() > kMaxParts) devlist.resize(kMaxParts);
  const int ndev = force_parts ? 1 : (int)devlist.size();
  int nparts = force_parts ? force_parts
                           : (ndev > 1 ? ndev : std::max(1, std::min(kMaxParts, env_int("SPLITPLAN_GRID_PARTS", 1))));
  nparts = (int)std::min<int64_t>(nparts, nchunks);
  const bool multi = ndev > 1 && nparts > 1;
  const bool separate = multi || (nparts > 1 && env_int("SPLITPLAN_GRID_SEPARATE", 0) != 0);
  // CTAs per partition: every partition placed on one device must be co-resident there
  int per_dev = nparts;
  if (multi) {
    per_dev = 1;
    for (int p = 0; p < nparts; ++p) {
      int c = 0;
      for (int r = 0; r < nparts; ++r) c += devlist[r] == devlist[p];
      per_dev = std::max(per_dev, c);
    }
  }
  int G = (int)std::min<int64_t>(resident / per_dev, (nchunks + nparts - 1) / nparts);
  G = std::max(G, 1);
  const int NC = (int)((nchunks + (int64_t)G * nparts - 1) / ((int64_t)G * nparts));
  G = (int)((nchunks + (int64_t)NC * nparts - 1) / ((int64_t)NC * nparts));
  const int64_t B = (int64_t)NC * grid_ch(mode);
  const int64_t line = 128 / (int64_t)vb;
  // halo: the widest read-back of any stage plus alignment slack, whole lines
  int64_t halo = 0;
  if (nparts > 1) {
    std::vector<StageShift> hs(L);
    int rc0 = check_cuda(cudaMemcpyAsync(hs.data(), shifts + lo, sizeof(StageShift) * L,
                                         cudaMemcpyDeviceToHost, st), "copy stage shifts");
    if (rc0) return rc0;
    rc0 = check_cuda(cudaStreamSynchronize(st), "sync");
    if (rc0) return rc0;
    int ms = 0;
    for (const StageShift& x : hs) ms = std::max(ms, std::max(std::max(x.i, x.id), std::max(x.s, x.su)));
    halo = ((int64_t)ms + 2 * line + line - 1) / line * line;
    if (halo > (int64_t)G * B) {  // the read-back spans a whole partition: no point splitting
      return run_grid_instance_parts(in, out, info, shifts, rv, reach, idx, inst, lo, L, ncol, mode, dyn,
                                     avail, st, 1);
    }
  }
  // one row buffer updated in place (a single launch whose stage shifts all
  // fit a one-neighbour halo): 1/3 of the row memory, L2-resident at cfg5.
  // Off by default (SPLITPLAN_GRID_INPLACE=1): with the reachable-frontier
  // skips the three-buffer kernel is faster at cfg5 (3.34 s vs 3.87 s,
  // profiles/r01/reach/cfg5_inplace_vs_3buf_reach.jsonl)
  int64_t inplace_hw = 0;
  if (nparts == 1 && !separate && env_int("SPLITPLAN_GRID_INPLACE", 0) != 0) {
    std::vector<StageShift> hs(L);
    int rc0 = check_cuda(cudaMemcpyAsync(hs.data(), shifts + lo, sizeof(StageShift) * L,
                                         cudaMemcpyDeviceToHost, st), "copy stage shifts");
    if (rc0) return rc0;
    rc0 = check_cuda(cudaStreamSynchronize(st), "sync");
    if (rc0) return rc0;
    int ms = 0;
    for (const StageShift& x : hs) ms = std::max(ms, std::max(std::max(x.i, x.id), std::max(x.s, x.su)));
    const int64_t hw = ((int64_t)ms + 16 / (int64_t)vb + line - 1) / line * line;
    if (hw <= B) inplace_hw = hw;
  }
  const bool inplace = inplace_hw > 0;
  const int64_t span = (grid_ch(mode) + line) + halo + G * B + line;
  const int64_t row_words = bp_row_words_for(mode, (int64_t)nparts * G * B);
  const size_t rows_bytes = inplace ? align_up(2 * (size_t)span * vb, 256) +
                                          align_up((size_t)G * 3 * 2 * (size_t)inplace_hw * vb, 256)
                                    : align_up(2 * kRowBufs * (size_t)span * vb, 256);
  const size_t ckpt_bytes = align_up(2 * (size_t)ncol * vb, 256);
  const size_t bp_stage = (size_t)row_words * 4;
  const size_t fixed = align_up((size_t)G * nparts * 4, 256) + 256 + nparts * rows_bytes;
  // segment length K: everything at once if it fits; else the longest
  // segments the workspace holds.  Segments are aligned to the END of the
  // chain and the last one keeps its back-pointers from the forward pass, so
  // the recompute costs L - K stages (2L - K in total), not L.
  int K = L;
  auto need = [&](int k) {
    const size_t nseg = (size_t)((L + k - 1) / k);
    return fixed + (k == L ? 2 : nseg + 1) * ckpt_bytes + align_up((size_t)k * bp_stage, 256);
  };
  const int force_k = env_int("SPLITPLAN_GRID_SEGMENT", 0);
  if (force_k > 0) K = std::min(force_k, L);
  if (need(K) > avail) {
    const size_t base = fixed + 2 * ckpt_bytes;
    K = avail > base ? (int)std::min<size_t>((size_t)L, (avail - base) / bp_stage) : 1;
    K = std::max(K, 1);
    while (K > 1 && need(K) > avail) K -= std::max(1, K / 64);
    if (need(K) > avail) {  // fall back to the smallest footprint, ~sqrt(L * ckpt / bp) stages
      K = (int)std::max<double>(1.0, std::sqrt((double)L * (double)ckpt_bytes / (double)bp_stage));
      K = std::min(K, L);
      while (K > 1 && need(K) > avail && need(K / 2) < need(K)) K /= 2;
    }
  }
  if (need(K) > avail) {
    set_required_workspace(need(K) + (avail > 0 ? 0 : 0) + (64 << 20));
    set_error(SP_ERR_WORKSPACE, "instance %lld (%d x %lld) needs %zu B of DP workspace, %zu B available",
              (long long)inst, L, (long long)ncol, need(K), avail);
    return SP_ERR_WORKSPACE;
  }
  Carve cv{dyn, avail};
  uint32_t* prog = (uint32_t*)cv.take((size_t)G * nparts * 4);
  int64_t* state = (int64_t*)cv.take(4 * sizeof(int64_t));
  uint8_t* rows[kMaxParts] = {};
  uint32_t* progs[kMaxParts] = {};
  const StageShift* pshifts[kMaxParts] = {};
  const int64_t* prv[kMaxParts] = {};
  const int2* preach[kMaxParts] = {};
  PeerParts peers;
  peers.cur = cur_dev;
  for (int p = 0; p < nparts; ++p) {
    peers.dev[p] = multi ? devlist[p] : peers.cur;
    pshifts[p] = shifts + lo;
    prv[p] = rv + lo;
    preach[p] = reach ? reach + lo : nullptr;
    if (peers.dev[p] == peers.cur) {
      rows[p] = (uint8_t*)cv.take(rows_bytes);
      progs[p] = prog + (size_t)p * G;
      continue;
    }
    rows[p] = (uint8_t*)peers.alloc(peers.dev[p], rows_bytes);
    progs[p] = (uint32_t*)peers.alloc(peers.dev[p], (size_t)G * 4);
    StageShift* sh_copy = (StageShift*)peers.alloc(peers.dev[p], sizeof(StageShift) * L);
    int64_t* rv_copy = (int64_t*)peers.alloc(peers.dev[p], sizeof(int64_t) * L);
    if (!rows[p] || !progs[p] || !sh_copy || !rv_copy) {
      set_error(SP_ERR_CUDA, "partition %d: device %d allocation failed", p, peers.dev[p]);
      return SP_ERR_CUDA;
    }
    int rc0 = check_cuda(cudaMemcpyPeerAsync(sh_copy, peers.dev[p], shifts + lo, peers.cur,
                                             sizeof(StageShift) * L, st), "copy stage records to peer");
    if (rc0) return rc0;
    rc0 = check_cuda(cudaMemcpyPeerAsync(rv_copy, peers.dev[p], rv + lo, peers.cur, sizeof(int64_t) * L, st),
                     "copy stage values to peer");
    if (rc0) return rc0;
    pshifts[p] = sh_copy;
    prv[p] = rv_copy;
    if (reach) {
      int2* reach_copy = (int2*)peers.alloc(peers.dev[p], sizeof(int2) * L);
      if (!reach_copy) {
        set_error(SP_ERR_CUDA, "partition %d: device %d allocation failed", p, peers.dev[p]);
        return SP_ERR_CUDA;
      }
      rc0 = check_cuda(cudaMemcpyPeerAsync(reach_copy, peers.dev[p], reach + lo, peers.cur, sizeof(int2) * L, st),
                       "copy reachable frontiers to peer");
      if (rc0) return rc0;
      preach[p] = reach_copy;
    }
  }
  if (multi) {  // every used device reaches every other one
    for (int p = 0; p < nparts; ++p)
      for (int r = 0; r < nparts; ++r) {
        if (peers.dev[p] == peers.dev[r]) continue;
        cudaSetDevice(peers.dev[p]);
        const cudaError_t e = cudaDeviceEnablePeerAccess(peers.dev[r], 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
          cudaSetDevice(peers.cur);
          return check_cuda(e, "cudaDeviceEnablePeerAccess");
        }
        cudaGetLastError();
      }
    cudaSetDevice(peers.cur);
  }
  if (separate) {
    int rc0 = check_cuda(cudaEventCreateWithFlags(&peers.start, cudaEventDisableTiming), "event");
    if (rc0) return rc0;
    for (int p = 0; p < nparts; ++p) {
      cudaSetDevice(peers.dev[p]);
      rc0 = check_cuda(cudaStreamCreateWithFlags(&peers.stream[p], cudaStreamNonBlocking), "partition stream");
      if (!rc0) rc0 = check_cuda(cudaEventCreateWithFlags(&peers.done[p], cudaEventDisableTiming), "event");
      cudaSetDevice(peers.cur);
      if (rc0) return rc0;
    }
  }
  const int nseg = (L + K - 1) / K;
  const int nckpt = K == L ? 2 : nseg + 1;
  std::vector<uint8_t*> ckpt(nckpt);
  for (int c = 0; c < nckpt; ++c) ckpt[c] = (uint8_t*)cv.take(ckpt_bytes);
  uint32_t* bp = (uint32_t*)cv.take((size_t)K * bp_stage);

  GridArgs g = {};
  g.shifts = shifts + lo;
  g.reach = reach ? reach + lo : nullptr;
  g.rv = rv + lo;
  g.ncol = (int)ncol;
  g.G = G;
  g.NC = NC;
  g.sac = 0;
  for (int p = 0; p < nparts; ++p) g.rows[p] = rows[p];
  g.nparts = nparts;
  g.part_base = 0;
  g.launch_parts = nparts;
  g.sys = (multi || env_int("SPLITPLAN_GRID_SYS", 0)) ? 1 : 0;
  g.halo = (int)halo;
  g.bp_row_words = row_words;
  for (int p = 0; p < nparts; ++p) g.progs[p] = progs[p];
  {
    uint8_t sac = 0;
    int rc = check_cuda(cudaMemcpyAsync(&sac, in->source_at_client + inst, 1, cudaMemcpyDeviceToHost, st),
                        "copy source_at_client");
    if (rc) return rc;
    rc = check_cuda(cudaStreamSynchronize(st), "sync");
    if (rc) return rc;
    g.sac = sac ? 1 : 0;
  }
  auto launch = [&](int k0, int cnt, const uint8_t* init, uint8_t* outrow, uint32_t* bpp) -> int {
    g.k_begin = k0;
    g.k_count = cnt;
    g.init_c = init;
    g.init_s = init ? init + ncol * vb : nullptr;
    g.out_c = outrow;
    g.out_s = outrow ? outrow + ncol * vb : nullptr;
    g.bp = bpp;
    // every partition's counters are zero before any partition starts
    zero_progs_kernel<<<1, 256, 0, st>>>(g);
    int rc = launch_check("zero_progs_kernel launch");
    if (rc) return rc;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (profiling()) {
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, st);
    }
    if (inplace) {
      GridInplaceArgs gi = {};
      gi.shifts = g.shifts;
      gi.reach = g.reach;
      gi.rv = g.rv;
      gi.k_begin = g.k_begin;
      gi.k_count = g.k_count;
      gi.ncol = g.ncol;
      gi.G = G;
      gi.NC = NC;
      gi.sac = g.sac;
      gi.hw = (int)inplace_hw;
      gi.init_c = g.init_c;
      gi.init_s = g.init_s;
      gi.out_c = g.out_c;
      gi.out_s = g.out_s;
      gi.bp = g.bp;
      gi.bp_row_words = g.bp_row_words;
      gi.prog = progs[0];
      gi.rows = rows[0];
      gi.halo = rows[0] + align_up(2 * (size_t)span * vb, 256);
      gi.row_hint = env_int("SPLITPLAN_ROW_EVICT_LAST", 0) ? 1 : 0;
      rc = launch_grid_inplace(mode, gi, st);
      if (rc) return rc;
    } else if (!separate) {
      rc = launch_grid(mode, g, st);
      if (rc) return rc;
    } else {  // one launch per partition, all in flight together
      rc = check_cuda(cudaEventRecord(peers.start, st), "record partition start");
      if (rc) return rc;
      for (int p = 0; p < nparts && !rc; ++p) {
        GridArgs gp = g;
        gp.part_base = p;
        gp.launch_parts = 1;
        gp.shifts = pshifts[p];
        gp.reach = preach[p];
        gp.rv = prv[p];
        cudaSetDevice(peers.dev[p]);
        rc = check_cuda(cudaStreamWaitEvent(peers.stream[p], peers.start, 0), "partition wait");
        if (!rc) rc = launch_grid(mode, gp, peers.stream[p]);
        if (!rc) rc = check_cuda(cudaEventRecord(peers.done[p], peers.stream[p]), "record partition end");
      }
      cudaSetDevice(peers.cur);
      if (rc) return rc;
      for (int p = 0; p < nparts; ++p) {
        rc = check_cuda(cudaStreamWaitEvent(st, peers.done[p], 0), "join partitions");
        if (rc) return rc;
      }
    }
    if (profiling()) {
      cudaEventRecord(e1, st);
      const double cells = (double)cnt * (double)ncol;
      prof_record_dp(e0, e1, cells, cells * (bpp ? hbm_bytes_per_cell(mode, DPV_SMEM) : 0.0), DPV_GRID);
    }
    return SP_OK;
  };
  int rc;
  // segment boundaries, aligned to the end: segment sg is [seg_begin(sg), seg_begin(sg + 1))
  auto seg_begin = [&](int sg) { return sg == 0 ? 0 : L - (nseg - sg) * K; };  // seg_begin(nseg) == L
  if (K == L) {
    rc = launch(0, L, nullptr, ckpt[1], bp);
    if (rc) return rc;
  } else {
    for (int sg = 0; sg < nseg; ++sg) {
      const int k0 = seg_begin(sg), cnt = seg_begin(sg + 1) - k0;
      rc = launch(k0, cnt, sg ? ckpt[sg] : nullptr, ckpt[sg + 1], sg + 1 == nseg ? bp : nullptr);
      if (rc) return rc;
    }
  }
  uint8_t* last = ckpt[K == L ? 1 : nseg];
  grid_end_kernel<<<1, 1, 0, st>>>(*in, info, inst, last, last + ncol * vb, state);
  rc = launch_check("grid_end_kernel launch");
  if (rc) return rc;
  int64_t hstate[3];
  rc = check_cuda(cudaMemcpyAsync(hstate, state, sizeof(hstate), cudaMemcpyDeviceToHost, st), "copy end state");
  if (rc) return rc;
  rc = check_cuda(cudaStreamSynchronize(st), "sync end state");
  if (rc) return rc;
  if (out && hstate[2] == 0) {
    if (K == L) {
      grid_backtrack_kernel<<<1, 1, 0, st>>>(*in, inst, shifts, bp, row_words, mode, 0, L, state, *out);
      rc = launch_check("grid_backtrack_kernel launch");
      if (rc) return rc;
    } else {
      for (int sg = nseg - 1; sg >= 0; --sg) {
        const int k0 = seg_begin(sg), cnt = seg_begin(sg + 1) - k0;
        if (sg + 1 < nseg) {  // the last segment's back-pointers are still there
          rc = launch(k0, cnt, sg ? ckpt[sg] : nullptr, nullptr, bp);
          if (rc) return rc;
        }
        grid_backtrack_kernel<<<1, 1, 0, st>>>(*in, inst, shifts, bp, row_words, mode, k0, cnt, state,
                                                *out);
        rc = launch_check("grid_backtrack_kernel launch");
        if (rc) return rc;
      }
    }
  }
  if (out) {
    grid_finish_kernel<<<1, 1, 0, st>>>(*in, inst, state, idx, *out);
    rc = launch_check("grid_finish_kernel launch");
    if (rc) return rc;
  }
  // the caller's next use of the workspace is stream-ordered after these
  return SP_OK;
}

// Shared driver of sp_plan_dp and sp_build_dp_tables.
int run_dp(const sp_instances* in, sp_policies* out, double* tab_c, double* tab_s, void* ws,
           size_t ws_bytes, cudaStream_t st, size_t* q_min = nullptr, size_t* q_full = nullptr) {
  const int64_t n = in->n, total = in->total_layers;
  if (n == 0) return SP_OK;
  Carve cv{(uint8_t*)ws, ws_bytes};
  InstInfo* info = (InstInfo*)cv.take(sizeof(InstInfo) * n);
  StageShift* shifts = (StageShift*)cv.take(sizeof(StageShift) * total);
  int64_t* rv = (int64_t*)cv.take(sizeof(int64_t) * total);
  int32_t* idx = (int32_t*)cv.take(sizeof(int32_t) * total);
  DpWork* work = (DpWork*)cv.take(sizeof(DpWork) * n);
  int2* reach = (int2*)cv.take(sizeof(int2) * total);
  const size_t fixed = align_up(cv.used, 256);
  if (!ws || fixed > ws_bytes) {
    set_required_workspace(fixed + (1 << 20));
    set_error(SP_ERR_WORKSPACE, "workspace %zu B < fixed part %zu B", ws_bytes, fixed);
    return SP_ERR_WORKSPACE;
  }
  const int grid = (int)std::min<int64_t>(n, 1 << 20);
  prep_kernel<<<grid, 128, 0, st>>>(*in, info, shifts, rv, reach);
  int rc = launch_check("prep_kernel launch");
  if (rc) return rc;

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

  const size_t avail = ws_bytes - fixed;
  uint8_t* dyn = (uint8_t*)ws + fixed;
  const int force = forced_variant();
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
  for (int64_t k = 0; k < n; ++k) {
    const int64_t ncol = hinfo[k].w_eff + 1;
    if (ncol > kMaxCols) {
      set_error(SP_ERR_UNSUPPORTED, "instance %lld: W_eff = %lld exceeds the supported 2^31 columns",
                (long long)k, (long long)hinfo[k].w_eff);
      return SP_ERR_UNSUPPORTED;
    }
    Item it;
    it.inst = k;
    it.L = hoff[k + 1] - hoff[k];
    it.ncol = ncol;
    it.mode = hinfo[k].mode;
    if (it.mode != cached_mode || ncol != cached_ncol || it.L != cached_L) {
      cached = plan_instance(it.mode, it.L, ncol, force, tab_c != nullptr);
      cached_mode = it.mode;
      cached_ncol = ncol;
      cached_L = it.L;
    }
    it.plan = cached;
    items.push_back(it);
  }

  if (q_min) {  // workspace query (sp_plan_dp_workspace_bytes): no DP launched
    size_t mn = 0, full = 0;
    for (const Item& it : items) {
      const bool grid = tab_c == nullptr && (force == DPV_GRID || it.ncol >= kGridMinCols);
      size_t imin = it.plan.bp + it.plan.rows, ifull = imin;
      if (grid) grid_workspace_bytes(it.mode, it.L, it.ncol, &imin, &ifull);
      mn = std::max(mn, imin);
      full = grid ? std::max(full, ifull) : full + ifull;
    }
    *q_min = fixed + mn;
    *q_full = fixed + std::max(full, mn);
    return SP_OK;
  }
  const int2* a_reach = env_int("SPLITPLAN_NO_REACH", 0) ? nullptr : reach;
  // instances too large for a wave (or wider than 4M columns) run alone over
  // the whole GPU (grid path, checkpointing if needed)
  {
    std::vector<Item> rest;
    rest.reserve(items.size());
    for (const Item& it : items) {
      const bool grid = tab_c == nullptr &&
                        (force == DPV_GRID || it.ncol >= kGridMinCols || it.plan.bp + it.plan.rows > avail);
      if (!grid) {
        rest.push_back(it);
        continue;
      }
      rc = run_grid_instance(in, out, info, shifts, rv, a_reach, idx, it.inst, hoff[it.inst], (int)it.L, it.ncol,
                             it.mode, dyn, avail, st);
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

  size_t pos = 0;
  std::vector<DpWork> hwork;
  struct Group {
    int mode;
    DpPlan plan;
    double cells = 0;
    std::vector<DpWork> items;
  };
  std::vector<Group> groups;
  while (pos < items.size()) {
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
    rc = check_cuda(cudaMemcpyAsync(work, hwork.data(), sizeof(DpWork) * hwork.size(),
                                    cudaMemcpyHostToDevice, st),
                    "upload work list");
    if (rc) return rc;
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
      rc = launch_plan(g.mode, g.plan, ga, cnt, st);
      if (rc) return rc;
      if (profiling()) {
        cudaEventRecord(e1, st);
        prof_record_dp(e0, e1, g.cells, g.cells * hbm_bytes_per_cell(g.mode, g.plan.variant),
                       g.plan.variant);
      }
      first += cnt;
    }
    if (out) {
      const int64_t nw = (int64_t)hwork.size();
      backtrack_kernel<<<(unsigned)((nw + 127) / 128), 128, 0, st>>>(*in, info, shifts, work, nw, dyn,
                                                                      idx, *out);
      rc = launch_check("backtrack_kernel launch");
      if (rc) return rc;
    }
    // the host work vector is reused next wave: the pageable H2D copy above is
    // synchronous with respect to the host buffer, so reuse is safe.
    pos = end;
  }
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

int sp_plan_dp_devices(const sp_instances* in, sp_policies* out, const int32_t* devices,
                       int32_t n_devices, void* ws, size_t ws_bytes, void* stream) {
  int rc = validate(in);
  if (rc) return rc;
  rc = validate_out(out);
  if (rc) return rc;
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
  for (int p = 0; p < n_devices; ++p)
    if (devices[p] < 0 || devices[p] >= count) {
      set_error(SP_ERR_INVALID, "devices[%d] = %d: no such device", p, devices[p]);
      return SP_ERR_INVALID;
    }
  tl_grid_devices.assign(devices, devices + n_devices);
  rc = run_dp(in, out, nullptr, nullptr, ws, ws_bytes, (cudaStream_t)stream);
  tl_grid_devices.clear();
  return rc;
}

int sp_build_dp_tables(const sp_instances* in, int64_t w_eff, double* client_table,
                       double* server_table, void* ws, size_t ws_bytes, void* stream) {
  int rc = validate(in);
  if (rc) return rc;
  if (in->n != 1 || !client_table || !server_table) {
    set_error(SP_ERR_INVALID, "sp_build_dp_tables takes exactly one instance and two tables");
    return SP_ERR_INVALID;
  }
  (void)w_eff;
  return run_dp(in, nullptr, client_table, server_table, ws, ws_bytes, (cudaStream_t)stream);
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
