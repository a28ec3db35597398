// Planner kernels of the B200 placement engine (reference: planner.py).
//
//   prep_kernel       per-instance W_eff, value domain, clamped stage shifts
//   dp_stage_kernel   K2: the two-state DP over the integer budget axis
//                     (planner.py:128-143) with a uint8 back-pointer per cell
//   backtrack_kernel  K3: end-side choice + pointer walk + _finish
//                     (planner.py:88-107, 146-202)
//   prefix_kernel     greedy / all-server / all-client (planner.py:205-225)
//   exhaustive_kernel plan_oracle (planner.py:228-268)
//   eq1_kernel        evaluator latency_of (evaluator.py:64-78)
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

// ---------------------------------------------------------------------------
// value domains

template <int MODE> struct VT;
template <> struct VT<VM_INT32> {
  using T = int32_t;
  static __device__ __forceinline__ T neg() { return INT32_MIN; }
};
template <> struct VT<VM_F64> {
  using T = double;
  static __device__ __forceinline__ T neg() { return -INFINITY; }
};
template <> struct VT<VM_F64_NAN> {
  using T = double;
  static __device__ __forceinline__ T neg() { return -INFINITY; }
};

__device__ __forceinline__ double to_f64(int32_t v, double g) {
  return v >= 0 ? dmul((double)v, g) : -INFINITY;
}
__device__ __forceinline__ double to_f64(double v, double) { return v; }

__device__ __forceinline__ uint64_t gcd_u64(uint64_t a, uint64_t b) {
  while (b) {
    uint64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}

// ---------------------------------------------------------------------------
// block reductions (128-thread prep blocks)

template <typename T, typename Op>
__device__ T block_reduce(T v, Op op, T* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  T r = sh[0];
  for (int w = 1; w < nw; ++w) r = op(r, sh[w]);
  __syncthreads();
  return r;
}

// ---------------------------------------------------------------------------
// W_eff only (planner.py:120-125)

__global__ void weff_kernel(sp_instances in, int64_t* w_eff) {
  __shared__ int64_t sh64[32];
  for (int64_t k = blockIdx.x; k < in.n; k += gridDim.x) {
    const int64_t lo = in.layer_off[k], hi = in.layer_off[k + 1];
    int64_t worst = 0;
    for (int64_t l = lo + threadIdx.x; l < hi; l += blockDim.x)
      worst += max(in.client_units[l] + in.down_units[l], in.server_units[l] + in.up_units[l]);
    worst = block_reduce(worst, [](int64_t a, int64_t b) { return a + b; }, sh64);
    if (threadIdx.x == 0) w_eff[k] = min(in.budget[k], worst);
  }
}

// ---------------------------------------------------------------------------
// prep: W_eff, value domain, clamped shifts, scaled values

__global__ void prep_kernel(sp_instances in, InstInfo* info, StageShift* shifts, int64_t* rv, int2* reach) {
  __shared__ int64_t sh64[32];
  __shared__ uint64_t shu[32];
  __shared__ int shi[32];
  for (int64_t k = blockIdx.x; k < in.n; k += gridDim.x) {
    const int64_t lo = in.layer_off[k], hi = in.layer_off[k + 1];
    int64_t worst = 0;
    int finite = 1, integral = 1;
    uint64_t isum = 0, g = 0;
    for (int64_t l = lo + threadIdx.x; l < hi; l += blockDim.x) {
      worst += max(in.client_units[l] + in.down_units[l], in.server_units[l] + in.up_units[l]);
      const double r = in.r[l];
      if (!isfinite(r)) {
        finite = 0;
      } else if (r != floor(r) || r >= 9007199254740992.0) {
        integral = 0;
      } else {
        const uint64_t v = (uint64_t)r;  // r >= 0 (problem.py:151-153)
        isum = min(isum + v, (uint64_t)1 << 62);
        g = gcd_u64(g, v);
      }
    }
    worst = block_reduce(worst, [](int64_t a, int64_t b) { return a + b; }, sh64);
    finite = block_reduce(finite, [](int a, int b) { return a & b; }, shi);
    integral = block_reduce(integral, [](int a, int b) { return a & b; }, shi);
    isum = block_reduce(isum, [](uint64_t a, uint64_t b) { return min(a + b, (uint64_t)1 << 62); }, shu);
    g = block_reduce(g, [](uint64_t a, uint64_t b) { return gcd_u64(a, b); }, shu);
    if (g == 0) g = 1;
    const int64_t W = min(in.budget[k], worst);
    int32_t mode;
    if (!finite) mode = VM_F64_NAN;
    else if (integral && isum < ((uint64_t)1 << 53) && isum / g <= (uint64_t)INT32_MAX) mode = VM_INT32;
    else mode = VM_F64;
    if (threadIdx.x == 0) {
      InstInfo r;
      r.w_eff = W;
      r.scale = (double)g;
      r.end_c = -INFINITY;
      r.end_s = -INFINITY;
      r.mode = mode;
      r.pad = 0;
      info[k] = r;
    }
    const int64_t cap = min(W + 1, kMaxCols);
    for (int64_t l = lo + threadIdx.x; l < hi; l += blockDim.x) {
      const int64_t i = in.client_units[l], s = in.server_units[l];
      const int64_t u = in.up_units[l], d = in.down_units[l];
      StageShift sh;
      sh.i = (int32_t)min(i, cap);
      sh.id = (int32_t)min(i + d, cap);
      sh.s = (int32_t)min(s, cap);
      sh.su = (int32_t)min(s + u, cap);
      shifts[l] = sh;
      const double r = in.r[l];
      if (mode == VM_INT32) {
        rv[l] = (int64_t)((uint64_t)r / g);
      } else {
        rv[l] = __double_as_longlong(r);
      }
    }
    // reachable frontier: the first column of row k of C and of S that holds a
    // reachable value (rows are monotone in j; every column below it is
    // unreachable, NEG-like).  reach[lo + k] describes the row stage k reads.
    // Not in the NaN domain, where "unreachable" cells may hold NaN.
    __syncthreads();  // the block's clamped shifts are in global memory
    if (threadIdx.x == 0 && reach) {
      const bool sac = in.source_at_client[k] != 0;
      int64_t mc = sac ? 0 : cap, ms = sac ? cap : 0;
      for (int64_t l = lo; l < hi; ++l) {
        reach[l] = mode == VM_F64_NAN ? make_int2(0, 0) : make_int2((int)min(mc, cap), (int)min(ms, cap));
        const StageShift sh = shifts[l];
        const int64_t nc = min(mc + sh.i, ms + sh.id), ns = min(ms + sh.s, mc + sh.su);
        mc = min(nc, cap);
        ms = min(ns, cap);
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K2: DP stage kernels
//
// One instance = two budget-indexed rows C and S (W_eff + 1 columns) updated
// once per layer k (planner.py:128-143):
//   C_k[j] = r_k + max(C_{k-1}[j - i_k], S_{k-1}[j - i_k - d_k])
//   S_k[j] =       max(S_{k-1}[j - s_k], C_{k-1}[j - s_k - u_k])
// Three variants hold the rows in different places:
//   * dp_stage_kernel<ROWS_SMEM=true>   one CTA, rows in its SMEM
//   * dp_cluster_kernel                 a thread-block cluster, rows split
//                                       across the CTAs' distributed SMEM
//   * dp_stage_kernel<ROWS_SMEM=false>  one CTA, rows in global memory
// Single-CTA variants update the rows IN PLACE, walking 32-aligned chunks of
// CH = E*T columns from the top down: a chunk computes its new cells into
// registers (its reads only touch columns <= its own, which no later chunk of
// this stage writes), then a barrier, then the writes.  Each row carries CH
// cells of NEG padding in front, and each chunk clamps the stage shifts to
// its top (shift' = min(shift, chunk_top)), so every read is a plain in-bounds
// load: shifted indices that were negative land in the padding and read NEG.
//
// Back-pointers are ballot-packed per warp: for each 32-column group one
// 32-bit word per flag -- C-stay, S-stay, and in the NaN-propagating domain
// also C-switch and S-switch.  The flags are exactly the predicates
// _backtrace evaluates (planner.py:159-178):
//   C-stay  : j>=i    and C[k-1][j-i]   + r == C[k][j]
//   C-switch: j>=i+d  and S[k-1][j-i-d] + r == C[k][j]
//   S-stay  : j>=s    and S[k-1][j-s]       == S[k][j]
//   S-switch: j>=s+u  and C[k-1][j-s-u]     == S[k][j]
// Outside the NaN domain a reachable cell that does not stay always switches
// (its value came from the other predecessor), so two words suffice.

struct DpArgs {
  const int64_t* layer_off;
  const uint8_t* sac;
  InstInfo* info;
  const StageShift* shifts;
  const int64_t* rv;
  const int2* reach;  // per stage: first reachable column of the C / S row it reads
  const DpWork* work;
  uint8_t* bp;
  uint8_t* rows;
  double* tab_c;  // optional full-table output (build_dp_tables), n == 1
  double* tab_s;
};

__host__ __device__ inline int bp_words(int mode) { return mode == VM_F64_NAN ? 4 : 2; }

struct CellFlags {
  bool c_stay, s_stay, c_sw, s_sw;
};

// One DP cell from its four predecessor values (NEG where the shifted column
// is negative).  v* tell whether each shifted column was >= 0; only the NaN
// domain needs them (elsewhere NEG can never reproduce a reachable value).
template <int MODE, typename V>
__device__ __forceinline__ CellFlags cell_update(V ca, V cb, V sa, V sb, V rk, bool vi, bool vid,
                                                 bool vs, bool vsu, V& cn, V& sn) {
  CellFlags f;
  if (MODE == VM_INT32) {
    // exact integer arithmetic: C-stay <=> ca >= cb, S-stay <=> sa >= sb
    f.c_stay = ca >= cb;
    f.s_stay = sa >= sb;
    cn = (f.c_stay ? ca : cb) + rk;
    sn = f.s_stay ? sa : sb;
    f.c_sw = !f.c_stay;
    f.s_sw = !f.s_stay;
  } else if (MODE == VM_F64) {
    const V cm = ca >= cb ? ca : cb;
    sn = sa >= sb ? sa : sb;
    cn = dadd(cm, rk);
    f.c_stay = dadd(ca, rk) == cn;  // fl(a + r) == C[k][j], not a >= b
    f.s_stay = sa == sn;
    f.c_sw = !f.c_stay;
    f.s_sw = !f.s_stay;
  } else {  // np.maximum propagates NaN
    const V cm = (ca != ca) ? ca : ((cb != cb) ? cb : (ca >= cb ? ca : cb));
    sn = (sa != sa) ? sa : ((sb != sb) ? sb : (sa >= sb ? sa : sb));
    cn = dadd(cm, rk);
    f.c_stay = vi && dadd(ca, rk) == cn;
    f.c_sw = vid && dadd(cb, rk) == cn;
    f.s_stay = vs && sa == sn;
    f.s_sw = vsu && sb == sn;
  }
  return f;
}

// warp-collective: pack the 32 lanes' flags of one column group into words
template <int MODE>
__device__ __forceinline__ void emit_bp(uint32_t* row_words, int group, int ngroups, CellFlags f,
                                        bool active) {
  const uint32_t m0 = __ballot_sync(0xffffffffu, active && f.c_stay);
  const uint32_t m1 = __ballot_sync(0xffffffffu, active && f.s_stay);
  if (MODE == VM_F64_NAN) {
    const uint32_t m2 = __ballot_sync(0xffffffffu, active && f.c_sw);
    const uint32_t m3 = __ballot_sync(0xffffffffu, active && f.s_sw);
    if ((threadIdx.x & 31) == 0 && group < ngroups)
      reinterpret_cast<uint4*>(row_words)[group] = make_uint4(m0, m1, m2, m3);
  } else {
    if ((threadIdx.x & 31) == 0 && group < ngroups)
      reinterpret_cast<uint2*>(row_words)[group] = make_uint2(m0, m1);
  }
}

// Materialise a pointer in a register so the compiler cannot re-associate
// (base + offset) + index into wide 64-bit index arithmetic per load: every
// predecessor load then costs one IMAD.WIDE.U32 on a chunk-uniform base.
template <typename T>
__device__ __forceinline__ const T* opaque(const T* p) {
  asm("" : "+l"(p));
  return p;
}

template <int MODE>
__device__ __forceinline__ void load_stage_tile(const DpArgs& a, int64_t lo, int k, int L,
                                                StageShift* st_sh, typename VT<MODE>::T* st_r) {
  using V = typename VT<MODE>::T;
  const int cnt = min(kStageTile, L - k);
  for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
    st_sh[t] = a.shifts[lo + k + t];
    const int64_t bits = a.rv[lo + k + t];
    if (MODE == VM_INT32) st_r[t] = (V)(int32_t)bits;
    else st_r[t] = (V)__longlong_as_double(bits);
  }
}

// Single-CTA kernel, T threads x E columns per chunk (CH = T*E), both
// template constants so every predecessor load is `LDS [base + imm]` on four
// chunk-uniform bases.  Rows hold CH cells of NEG padding in front and are
// padded at the end to whole chunks (nch*CH columns), so no load, store or
// back-pointer word needs a bounds check: cells past W_eff compute garbage
// that no valid cell ever reads (reads only go left), and their back-pointer
// bits are never visited.  bp rows are nch*CH/32 groups wide.
template <int MODE, bool ROWS_SMEM, int T, int E>
__global__ void __launch_bounds__(T, (T >= 1024 ? 1 : 1024 / T)) dp_stage_kernel(DpArgs a) {
  using V = typename VT<MODE>::T;
  constexpr int CH = T * E;
  extern __shared__ __align__(16) unsigned char smem[];
  StageShift* st_sh = reinterpret_cast<StageShift*>(smem);
  V* st_r = reinterpret_cast<V*>(smem + kStageTile * sizeof(StageShift));
  const size_t stage_bytes = align_up(kStageTile * (sizeof(StageShift) + sizeof(V)), 16);

  const DpWork wk = a.work[blockIdx.x];
  const int64_t inst = wk.inst;
  const int64_t lo = a.layer_off[inst];
  const int L = (int)(a.layer_off[inst + 1] - lo);
  const int ncol = (int)(a.info[inst].w_eff + 1);
  const double g = a.info[inst].scale;
  const bool sac = a.sac[inst] != 0;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int nch = (ncol + CH - 1) / CH;
  const int span = CH + nch * CH;
  const int64_t row_words = wk.bp_row_words;

  V* base = ROWS_SMEM ? reinterpret_cast<V*>(smem + stage_bytes)
                      : reinterpret_cast<V*>(a.rows + wk.row_off);
  V* Cp = base + CH;         // C row, column 0
  V* Sp = base + span + CH;  // S row, column 0
  const V NEG = VT<MODE>::neg();
  const V ZERO = V(0);

  for (int x = tid - CH; x < nch * CH; x += T) {
    Cp[x] = (x >= 0 && x < ncol && sac) ? ZERO : NEG;
    Sp[x] = (x >= 0 && x < ncol && !sac) ? ZERO : NEG;
    if (a.tab_c && x >= 0 && x < ncol) {
      a.tab_c[x] = sac ? 0.0 : -INFINITY;
      a.tab_s[x] = sac ? -INFINITY : 0.0;
    }
  }

  uint32_t* bpw = reinterpret_cast<uint32_t*>(a.bp + wk.bp_off);
  for (int k = 0; k < L; ++k) {
    const int kt = k % kStageTile;
    if (kt == 0) {
      __syncthreads();
      load_stage_tile<MODE>(a, lo, k, L, st_sh, st_r);
    }
    __syncthreads();
    const StageShift sh = st_sh[kt];
    const V rk = st_r[kt];
    uint32_t* bprow = bpw + (int64_t)k * row_words + warp * bp_words(MODE);

    for (int c = nch - 1; c >= 0; --c) {
      const int c0 = c * CH, ctop = c0 + CH;
      // chunk-uniform clamped shifts: every read stays in [-CH, nch*CH)
      const V* pca = Cp - min(sh.i, ctop) + c0 + tid;
      const V* pcb = Sp - min(sh.id, ctop) + c0 + tid;
      const V* psa = Sp - min(sh.s, ctop) + c0 + tid;
      const V* psb = Cp - min(sh.su, ctop) + c0 + tid;
      uint32_t* bpc = bprow + (c0 >> 5) * bp_words(MODE);
      V cn[E], sn[E];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int j = c0 + e * T + tid;
        const CellFlags f = cell_update<MODE, V>(pca[e * T], pcb[e * T], psa[e * T], psb[e * T], rk,
                                                 j >= sh.i, j >= sh.id, j >= sh.s, j >= sh.su,
                                                 cn[e], sn[e]);
        emit_bp<MODE>(bpc + e * (T / 32) * bp_words(MODE), 0, 1, f, true);
      }
      __syncthreads();
      V* qc = Cp + c0 + tid;
      V* qs = Sp + c0 + tid;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        qc[e * T] = cn[e];
        qs[e * T] = sn[e];
      }
      if (a.tab_c) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int j = c0 + e * T + tid;
          if (j < ncol) {
            a.tab_c[(int64_t)(k + 1) * ncol + j] = to_f64(cn[e], g);
            a.tab_s[(int64_t)(k + 1) * ncol + j] = to_f64(sn[e], g);
          }
        }
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    a.info[inst].end_c = to_f64(Cp[ncol - 1], g);
    a.info[inst].end_s = to_f64(Sp[ncol - 1], g);
  }
}

// ---------------------------------------------------------------------------
// K2 cluster variant: rows too long for one SM live in the distributed shared
// memory of a thread-block cluster of G CTAs (G <= 16).  CTA q owns columns
// [q*B, (q+1)*B) of both rows (B a multiple of 32), double-buffered (stage k
// reads buffer k&1 and writes buffer (k&1)^1), so one cluster barrier per
// stage orders everything: it releases this stage's writes and guarantees no
// CTA still reads the buffer the next stage overwrites.  Predecessor values
// come from whichever CTA owns the shifted column via ld.shared::cluster.
// Only the packed back-pointer words reach HBM.

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t cluster_addr(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ int32_t ld_cluster(uint32_t addr, int32_t) {
  int32_t v;
  asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ double ld_cluster(uint32_t addr, double) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

struct ClusterGeom {
  int G;          // CTAs per instance
  int B;          // columns owned per CTA (multiple of 32)
  uint32_t magic; // owner(x) = umulhi(x, magic) == x / B for x < G * B
};

template <int MODE>
__global__ void __launch_bounds__(kMaxThreads, 1) dp_cluster_kernel(DpArgs a, ClusterGeom geo) {
  using V = typename VT<MODE>::T;
  extern __shared__ __align__(16) unsigned char smem[];
  StageShift* st_sh = reinterpret_cast<StageShift*>(smem);
  V* st_r = reinterpret_cast<V*>(smem + kStageTile * sizeof(StageShift));
  const size_t stage_bytes = align_up(kStageTile * (sizeof(StageShift) + sizeof(V)), 16);
  V* rows = reinterpret_cast<V*>(smem + stage_bytes);  // [buf][C|S][B]

  const int G = geo.G, B = geo.B;
  const int q = (int)cluster_rank();
  const DpWork wk = a.work[blockIdx.x / G];
  const int64_t inst = wk.inst;
  const int64_t lo = a.layer_off[inst];
  const int L = (int)(a.layer_off[inst + 1] - lo);
  const int ncol = (int)(a.info[inst].w_eff + 1);
  const double g = a.info[inst].scale;
  const bool sac = a.sac[inst] != 0;
  const int T = blockDim.x, tid = threadIdx.x, warp = tid >> 5;
  const int j0 = q * B;
  const int jn = max(0, min(ncol, j0 + B) - j0);
  const int group_end = (j0 + jn + 31) >> 5;  // this CTA's back-pointer groups end here
  const int64_t row_words = wk.bp_row_words;
  const V NEG = VT<MODE>::neg();
  const V ZERO = V(0);
  const uint32_t rows_sa = smem_addr(rows);

  for (int t = tid; t < jn; t += T) {
    rows[t] = sac ? ZERO : NEG;      // buf 0, C
    rows[B + t] = sac ? NEG : ZERO;  // buf 0, S
    if (a.tab_c) {
      a.tab_c[j0 + t] = sac ? 0.0 : -INFINITY;
      a.tab_s[j0 + t] = sac ? -INFINITY : 0.0;
    }
  }
  // shared::cluster address of `rows` in every rank.  The window is linear in
  // the rank on sm_100 (base + r * stride); verify that once and keep a table
  // in SMEM as the fallback, so the inner loop never issues mapa (ADU pipe).
  __shared__ uint32_t rank_base[16];
  __shared__ int linear_ok;
  if (tid < G) rank_base[tid] = cluster_addr(rows_sa, (uint32_t)tid);
  __syncthreads();
  if (tid == 0) {
    int ok = 1;
    const uint32_t stride = G > 1 ? rank_base[1] - rank_base[0] : 0;
    for (int r = 0; r < G; ++r) ok &= rank_base[r] == rank_base[0] + (uint32_t)r * stride;
    linear_ok = ok;
  }
  __syncthreads();
  const bool linear = linear_ok != 0;
  const uint32_t base0 = rank_base[0];
  // per-rank step in the linear formula, net of the B columns a rank covers
  const uint32_t rank_step = (G > 1 ? rank_base[1] - rank_base[0] : 0) - (uint32_t)(B * sizeof(V));
  uint32_t* bpw = reinterpret_cast<uint32_t*>(a.bp + wk.bp_off);
  cluster_barrier();
  // the stage loop, instantiated once per addressing scheme (uniform branch)
  auto stages = [&](auto lin_tag) {
    constexpr bool LIN = decltype(lin_tag)::value;
    // predecessor value of row `rs` (0 = C, 1 = S) in buffer `buf` at global column x
    auto fetch = [&](int x0, uint32_t rowoff) -> V {
      const int x = max(x0, 0);  // branch-free: load a valid cell, select NEG below
      const uint32_t owner = __umulhi((uint32_t)x, geo.magic);
      const uint32_t rel = rowoff + (uint32_t)x * sizeof(V);
      uint32_t addr;
      if (LIN) addr = base0 + owner * rank_step + rel;
      else addr = rank_base[owner] + rel - owner * (uint32_t)(B * sizeof(V));
      const V v = ld_cluster(addr, V());
      return x0 >= 0 ? v : NEG;
    };
    for (int k = 0; k < L; ++k) {
      const int kt = k % kStageTile;
      if (kt == 0) {
        load_stage_tile<MODE>(a, lo, k, L, st_sh, st_r);
        __syncthreads();
      }
      const StageShift sh = st_sh[kt];
      const V rk = st_r[kt];
      const int cur = k & 1;
      const uint32_t offC = (uint32_t)((cur * 2 + 0) * B * (int)sizeof(V));
      const uint32_t offS = (uint32_t)((cur * 2 + 1) * B * (int)sizeof(V));
      V* Cn = rows + ((cur ^ 1) * 2 + 0) * B;
      V* Sn = rows + ((cur ^ 1) * 2 + 1) * B;
      uint32_t* bprow = bpw + (int64_t)k * row_words;
      constexpr int U = 4;
      for (int t0 = 0; t0 < jn; t0 += U * T) {  // warp-uniform trip count
        V ca[U], cb[U], sa[U], sb[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int t = t0 + u * T + tid;
          const int j = j0 + (t < jn ? t : 0);
          ca[u] = fetch(j - sh.i, offC);
          cb[u] = fetch(j - sh.id, offS);
          sa[u] = fetch(j - sh.s, offS);
          sb[u] = fetch(j - sh.su, offC);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int t = t0 + u * T + tid;
          const bool active = t < jn;
          const int j = j0 + t;
          V cn, sn;
          const CellFlags f = cell_update<MODE, V>(ca[u], cb[u], sa[u], sb[u], rk, j >= sh.i,
                                                   j >= sh.id, j >= sh.s, j >= sh.su, cn, sn);
          // groups past this CTA's columns belong to the next rank: never store them
          emit_bp<MODE>(bprow, (j0 + t0 + u * T) / 32 + warp, group_end, f, active);
          if (active) {
            Cn[t] = cn;
            Sn[t] = sn;
            if (a.tab_c) {
              a.tab_c[(int64_t)(k + 1) * ncol + j] = to_f64(cn, g);
              a.tab_s[(int64_t)(k + 1) * ncol + j] = to_f64(sn, g);
            }
          }
        }
      }
      cluster_barrier();
    }
  };
  if (linear) stages(std::true_type{});
  else stages(std::false_type{});
  // the CTA owning column ncol-1 publishes the end cell (buffer L & 1)
  if (tid == 0 && ncol - 1 >= j0 && ncol - 1 < j0 + B) {
    const int t = ncol - 1 - j0, buf = L & 1;
    a.info[inst].end_c = to_f64(rows[(buf * 2 + 0) * B + t], g);
    a.info[inst].end_s = to_f64(rows[(buf * 2 + 1) * B + t], g);
  }
  cluster_barrier();  // keep every CTA's SMEM alive until remote reads are done
}

// ---------------------------------------------------------------------------
// K2 cooperative variant: a cluster of G CTAs shares one instance whose rows
// live in global memory, double-buffered and sized so the rows of all
// co-resident instances stay in L2.  CTA q computes the columns
// [q*B, (q+1)*B) of the next buffer from any column of the current one; one
// cluster barrier (release/acquire, which also invalidates L1) per stage.
// Rows carry CH cells of NEG padding in front, and shifts are clamped per
// chunk exactly as in dp_stage_kernel, so reads need no bounds checks.

template <int MODE, int E>
__global__ void __launch_bounds__(kStageThreads, 2) dp_coop_kernel(DpArgs a, ClusterGeom geo) {
  using V = typename VT<MODE>::T;
  extern __shared__ __align__(16) unsigned char smem[];
  StageShift* st_sh = reinterpret_cast<StageShift*>(smem);
  V* st_r = reinterpret_cast<V*>(smem + kStageTile * sizeof(StageShift));

  const int G = geo.G, B = geo.B;
  const int q = (int)cluster_rank();
  const DpWork wk = a.work[blockIdx.x / G];
  const int64_t inst = wk.inst;
  const int64_t lo = a.layer_off[inst];
  const int L = (int)(a.layer_off[inst + 1] - lo);
  const int ncol = (int)(a.info[inst].w_eff + 1);
  const double g = a.info[inst].scale;
  const bool sac = a.sac[inst] != 0;
  const int T = blockDim.x, tid = threadIdx.x, warp = tid >> 5;
  const int CH = E * T;
  const int span = CH + ncol;
  const int j0 = q * B;
  const int jend = min(ncol, j0 + B);
  const int jn = max(0, jend - j0);
  const int group_end = (jend + 31) >> 5;
  const int64_t row_words = wk.bp_row_words;
  const V NEG = VT<MODE>::neg();
  const V ZERO = V(0);
  V* base = reinterpret_cast<V*>(a.rows + wk.row_off);  // [buf][C|S][CH pad + ncol]
  auto row = [&](int buf, int rs) { return base + (int64_t)(buf * 2 + rs) * span + CH; };

  for (int buf = 0; buf < 2; ++buf) {
    V* Cb = row(buf, 0);
    V* Sb = row(buf, 1);
    if (q == 0)
      for (int x = tid - CH; x < 0; x += T) Cb[x] = Sb[x] = NEG;  // padding, never rewritten
    if (buf == 0)
      for (int j = j0 + tid; j < jend; j += T) {
        Cb[j] = sac ? ZERO : NEG;
        Sb[j] = sac ? NEG : ZERO;
        if (a.tab_c) {
          a.tab_c[j] = sac ? 0.0 : -INFINITY;
          a.tab_s[j] = sac ? -INFINITY : 0.0;
        }
      }
  }
  uint32_t* bpw = reinterpret_cast<uint32_t*>(a.bp + wk.bp_off);
  cluster_barrier();
  for (int k = 0; k < L; ++k) {
    const int kt = k % kStageTile;
    if (kt == 0) {
      load_stage_tile<MODE>(a, lo, k, L, st_sh, st_r);
      __syncthreads();
    }
    const StageShift sh = st_sh[kt];
    const V rk = st_r[kt];
    const int cur = k & 1;
    const V* Cc = row(cur, 0);
    const V* Sc = row(cur, 1);
    V* Cn = row(cur ^ 1, 0);
    V* Sn = row(cur ^ 1, 1);
    uint32_t* bprow = bpw + (int64_t)k * row_words;
    for (int c0 = j0; c0 < jend; c0 += CH) {  // warp-uniform trip count
      const int ctop = c0 + CH;
      // chunk-uniform bases such that base + jr (jr >= c0 >= 0, unsigned) is the
      // clamped predecessor: one IMAD.WIDE.U32 per load
      const V* pca = opaque(Cc - min(sh.i, ctop));
      const V* pcb = opaque(Sc - min(sh.id, ctop));
      const V* psa = opaque(Sc - min(sh.s, ctop));
      const V* psb = opaque(Cc - min(sh.su, ctop));
      V ca[E], cb[E], sa[E], sb[E];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int j = c0 + e * T + tid;
        const uint32_t jr = (uint32_t)(j < jend ? j : jend - 1);
        ca[e] = pca[jr];
        cb[e] = pcb[jr];
        sa[e] = psa[jr];
        sb[e] = psb[jr];
      }
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int j = c0 + e * T + tid;
        const bool active = j < jend;
        V cn, sn;
        const CellFlags f = cell_update<MODE, V>(ca[e], cb[e], sa[e], sb[e], rk, j >= sh.i,
                                                 j >= sh.id, j >= sh.s, j >= sh.su, cn, sn);
        emit_bp<MODE>(bprow, (c0 + e * T) / 32 + warp, group_end, f, active);
        if (active) {
          Cn[(uint32_t)j] = cn;
          Sn[(uint32_t)j] = sn;
          if (a.tab_c) {
            a.tab_c[(int64_t)(k + 1) * ncol + j] = to_f64(cn, g);
            a.tab_s[(int64_t)(k + 1) * ncol + j] = to_f64(sn, g);
          }
        }
      }
    }
    cluster_barrier();
  }
  if (tid == 0 && ncol - 1 >= j0 && ncol - 1 < jend) {
    a.info[inst].end_c = to_f64(row(L & 1, 0)[ncol - 1], g);
    a.info[inst].end_s = to_f64(row(L & 1, 1)[ncol - 1], g);
  }
}

// ---------------------------------------------------------------------------
// K2 streaming variant (rows longer than one SM's shared memory): a cluster
// of G CTAs shares one instance, CTA q owning NC chunks of CH = T*E columns.
// The rows live in global memory, TRIPLE-buffered, sized so the rows of every
// co-resident instance stay in L2.  Each CTA is warp-specialised:
//   * one producer warp fetches, for every chunk, the four predecessor windows
//     (C at i, S at i+d, S at s, C at s+u; CH values + 128 B, 128-B aligned)
//     with the bulk-copy engine (cp.async.bulk, completion on a `full`
//     mbarrier) into an NSLOT-deep ring of shared-memory slots;
//   * T compute threads read them with conflict-free LDS like the single-CTA
//     kernel, store the new cells straight to the next row buffer (coalesced
//     warp stores) and the back-pointer words with an L2 evict-first policy,
//     and release the slot on its `empty` mbarrier.
// Stages are ordered by per-CTA progress counters in shared memory, read by
// the other CTAs of the cluster through DSMEM, instead of a cluster-wide
// barrier: stage s reads row s-1 from buffer (s-1)%3 and writes row s to
// buffer s%3, so the producer of CTA q may start stage s once every CTA at or
// left of q finished stage s-1 (all reads go left: shifts are >= 0) and every
// CTA finished stage s-2 (the last reader of the buffer stage s overwrites).
// CTAs therefore run up to one stage apart and the bulk copies of the next
// stage overlap the tail of the current one.

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void named_barrier(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ uint32_t ld_cluster_relaxed(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.relaxed.cluster.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void st_cluster_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.cluster.shared::cta.u32 [%0], %1;" ::"r"(smem_addr(p)), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_cluster() {
  asm volatile("fence.acq_rel.cluster;" ::: "memory");
}
__device__ __forceinline__ uint64_t evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void st_hint(int32_t* p, int32_t v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_hint(double* p, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.b64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void st_bp_words(uint32_t* p, uint32_t a, uint32_t b, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.b32 [%0], {%1, %2}, %3;" ::"l"(p), "r"(a), "r"(b), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st_bp_words(uint32_t* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d,
                                            uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(a), "r"(b),
               "r"(c), "r"(d), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void discard_l2(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

// warp-collective back-pointer emission with an L2 evict-first store
template <int MODE>
__device__ __forceinline__ void emit_bp_stream(uint32_t* words, CellFlags f, uint64_t pol) {
  const uint32_t m0 = __ballot_sync(0xffffffffu, f.c_stay);
  const uint32_t m1 = __ballot_sync(0xffffffffu, f.s_stay);
  if (MODE == VM_F64_NAN) {
    const uint32_t m2 = __ballot_sync(0xffffffffu, f.c_sw);
    const uint32_t m3 = __ballot_sync(0xffffffffu, f.s_sw);
    if ((threadIdx.x & 31) == 0) st_bp_words(words, m0, m1, m2, m3, pol);
  } else {
    if ((threadIdx.x & 31) == 0) st_bp_words(words, m0, m1, pol);
  }
}

struct StreamGeom {
  int G;         // CTAs per instance (cluster size)
  int NC;        // chunks per CTA
  int n_items;   // instances of the launch (set at launch)
  int row_hint;  // L2 policy of the row stores (set at launch)
  int diag;      // diagnostics only (SPLITPLAN_STREAM_DIAG; results are wrong when set):
                 // bit 0 skips the stage waits, bit 1 skips the window copies
  int cfg;       // kStreamCfgs index (host side)
};

constexpr int kRowBufs = 3;

// values of NEG padding in front of a streamed row: one chunk plus one 128-B
// line, so every window start (>= -CH) rounded down to 16 B stays in the row
// and every CTA block starts on a 128-B line
template <typename V, int CH>
__host__ __device__ constexpr int stream_pad() { return CH + 128 / (int)sizeof(V); }

// NI instances share one cluster and alternate stage by stage (A0 B0 A1 B1
// ...): while the producer waits for the other CTAs to finish instance A's
// stage k, the compute warps work through instance B's stage k, so the
// stage synchronisation latency overlaps useful work.
template <int MODE, int T, int E, int NSLOT, int NI, int NBUF>
__global__ void __launch_bounds__(T + 32, 2) dp_stream_kernel(DpArgs a, StreamGeom geo) {
  using V = typename VT<MODE>::T;
  constexpr int CH = T * E;
  constexpr int AL = 16 / (int)sizeof(V);        // values per 16 B
  constexpr int WIN = CH + AL;                    // values per staged window
  constexpr int PAD = stream_pad<V, CH>();
  constexpr int LINE = 128 / (int)sizeof(V);      // values per 128-B line
  constexpr int NWARP = T / 32;                   // compute warps
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + NSLOT;
  uint32_t* prog = reinterpret_cast<uint32_t*>(empty + NSLOT);  // [NI] stages completed
  V* slots = reinterpret_cast<V*>(smem + 256);                    // [NSLOT][4][WIN]
  V* negwin = slots + NSLOT * 4 * WIN;                             // [WIN] of NEG: windows below the frontier

  const int G = geo.G, NC = geo.NC;
  const int q = (int)cluster_rank();
  const int first = (int)(blockIdx.x / G) * NI;
  const int ni = min(NI, geo.n_items - first);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int B = NC * CH;
  const int j0 = q * B;
  const int64_t span = (int64_t)PAD + (int64_t)G * B + LINE;
  const V NEG = VT<MODE>::neg();
  const V ZERO = V(0);
  int64_t inst[NI], lo[NI], row_words[NI];
  int L[NI], ncol[NI];
  V* base[NI];
  int maxL = 0;
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    const DpWork wk = a.work[first + min(i, ni - 1)];
    inst[i] = wk.inst;
    lo[i] = a.layer_off[wk.inst];
    L[i] = i < ni ? (int)(a.layer_off[wk.inst + 1] - lo[i]) : 0;
    ncol[i] = (int)(a.info[wk.inst].w_eff + 1);
    base[i] = reinterpret_cast<V*>(a.rows + wk.row_off);  // [buf][C|S][PAD + G*B + LINE]
    row_words[i] = wk.bp_row_words;
    maxL = max(maxL, L[i]);
  }
  auto row = [&](int i, int buf, int rs) { return base[i] + (int64_t)(buf * 2 + rs) * span + PAD; };

  for (int i = 0; i < ni; ++i) {
    const bool sac = a.sac[inst[i]] != 0;
    for (int buf = 0; buf < NBUF; ++buf) {
      V* Cb = row(i, buf, 0);
      V* Sb = row(i, buf, 1);
      if (q == 0)
        for (int x = tid - PAD; x < 0; x += blockDim.x) Cb[x] = Sb[x] = NEG;  // never rewritten
      if (q == G - 1)
        for (int x = G * B + tid; x < G * B + LINE; x += blockDim.x) Cb[x] = Sb[x] = NEG;
      if (buf == 0)
        for (int j = j0 + tid; j < j0 + B; j += blockDim.x) {
          const bool valid = j < ncol[i];
          Cb[j] = (valid && sac) ? ZERO : NEG;
          Sb[j] = (valid && !sac) ? ZERO : NEG;
          if (a.tab_c && valid) {
            a.tab_c[j] = sac ? 0.0 : -INFINITY;
            a.tab_s[j] = sac ? -INFINITY : 0.0;
          }
        }
    }
  }
  for (int x = tid; x < WIN; x += blockDim.x) negwin[x] = NEG;
  if (tid == 0) {
    for (int b = 0; b < NSLOT; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], NWARP);
    }
    for (int i = 0; i < NI; ++i) prog[i] = 0;
    fence_mbar_init();
  }
  fence_proxy_async_global();
  __threadfence();
  cluster_barrier();  // rows initialised, barriers and counters live in every CTA

  if (warp == NWARP) {
    // ---------------- producer warp ----------------
    // lane o watches CTA o's progress counters (G <= 16 <= 32 lanes)
    const uint32_t my_prog = lane < G ? cluster_addr(smem_addr(prog), (uint32_t)lane) : 0u;
    uint32_t u = 0;
    for (int k = 0; k < maxL; ++k) {  // stage k of each instance in turn
      for (int i = 0; i < ni; ++i) {
        if (k >= L[i]) continue;
        const StageShift sh = a.shifts[lo[i] + k];  // issued before the wait: latency overlaps it
        const int2 rch = a.reach ? a.reach[lo[i] + k] : make_int2(0, 0);  // first reachable columns of C_k, S_k
        // every CTA <= q finished stage k (row k ready); WAR on the buffer this
        // stage overwrites: with 3 buffers every CTA finished k-1, with 2 every CTA k
        const uint32_t need =
            lane < G ? (uint32_t)(lane <= q || NBUF == 2 ? k : max(k - 1, 0)) : 0u;
        while (!(geo.diag & 1) &&
               !__all_sync(0xffffffffu, lane >= G || ld_cluster_relaxed(my_prog + 4u * i) >= need)) {
        }
        if (lane == 0) {
          fence_acq_rel_cluster();
          fence_proxy_async_global();
          const V* Cc = row(i, k % NBUF, 0);
          const V* Sc = row(i, k % NBUF, 1);
          const V* src[4] = {Cc, Sc, Sc, Cc};
          const int shf[4] = {sh.i, sh.id, sh.s, sh.su};
          for (int c = 0; c < NC; ++c, ++u) {
            const int slot = (int)(u % NSLOT);
            mbar_wait(&empty[slot], ((u / NSLOT) & 1) ^ 1);
            const int c0 = j0 + c * CH, ctop = c0 + CH;
            if (geo.diag & 2) {
              mbar_arrive(&full[slot]);
              continue;
            }
            // a window entirely below its row's reachable frontier is all NEG:
            // no copy, the compute warps read the NEG window instead
            int start[4];
            uint32_t ncopy = 0;
#pragma unroll
            for (int w = 0; w < 4; ++w) {
              start[w] = c0 - min(shf[w], ctop);
              ncopy += start[w] + CH > ((w == 0 || w == 3) ? rch.x : rch.y) ? 1u : 0u;
            }
            mbar_expect_tx(&full[slot], ncopy * WIN * sizeof(V));
#pragma unroll
            for (int w = 0; w < 4; ++w)
              if (start[w] + CH > ((w == 0 || w == 3) ? rch.x : rch.y))
                bulk_g2s(slots + (slot * 4 + w) * WIN, src[w] + (start[w] & ~(AL - 1)), WIN * sizeof(V),
                         &full[slot]);
          }
        }
        __syncwarp();
      }
    }
  } else {
    // ---------------- compute warps ----------------
    const uint64_t pol = evict_first_policy();
    // the rows are re-read next stage: keep them in L2 ahead of the streamed
    // back-pointers (geo.row_hint 0: normal, 1: evict_last)
    const uint64_t rpol = evict_last_policy();
    uint32_t u = 0;
    for (int k = 0; k < maxL; ++k) {
      for (int i = 0; i < ni; ++i) {
        if (k >= L[i]) continue;
        const StageShift sh = a.shifts[lo[i] + k];
        const int2 rch = a.reach ? a.reach[lo[i] + k] : make_int2(0, 0);
        // every cell of row k+1 below both frontiers is unreachable
        const int64_t next_front = a.reach ? min(min((int64_t)rch.x + sh.i, (int64_t)rch.y + sh.id),
                                                 min((int64_t)rch.y + sh.s, (int64_t)rch.x + sh.su))
                                           : 0;
        const int64_t rbits = a.rv[lo[i] + k];
        const V rk = MODE == VM_INT32 ? (V)(int32_t)rbits : (V)__longlong_as_double(rbits);
        V* Cn = row(i, (k + 1) % NBUF, 0);
        V* Sn = row(i, (k + 1) % NBUF, 1);
        const DpWork wk = a.work[first + i];
        uint32_t* bprow = reinterpret_cast<uint32_t*>(a.bp + wk.bp_off) + (int64_t)k * row_words[i] +
                          warp * bp_words(MODE);
        for (int c = 0; c < NC; ++c, ++u) {
          const int slot = (int)(u % NSLOT);
          const int c0 = j0 + c * CH, ctop = c0 + CH;
          const V* ws = slots + slot * 4 * WIN + tid;
          const int sa = c0 - min(sh.i, ctop), sb = c0 - min(sh.id, ctop);
          const int sc = c0 - min(sh.s, ctop), sd = c0 - min(sh.su, ctop);
          // windows below the reachable frontier were not copied: read NEG
          const V* pca = (sa + CH > rch.x ? ws + 0 * WIN : negwin + tid) + (sa & (AL - 1));
          const V* pcb = (sb + CH > rch.y ? ws + 1 * WIN : negwin + tid) + (sb & (AL - 1));
          const V* psa = (sc + CH > rch.y ? ws + 2 * WIN : negwin + tid) + (sc & (AL - 1));
          const V* psb = (sd + CH > rch.x ? ws + 3 * WIN : negwin + tid) + (sd & (AL - 1));
          uint32_t* bpc = bprow + (c0 >> 5) * bp_words(MODE);
          mbar_wait(&full[slot], (u / NSLOT) & 1);
          V cn[E], sn[E];
          if ((int64_t)ctop <= next_front && !a.tab_c) {  // whole chunk unreachable: NEG, no back-pointers
#pragma unroll
            for (int e = 0; e < E; ++e) cn[e] = sn[e] = NEG;
          } else {
#pragma unroll
            for (int e = 0; e < E; ++e) {
              const int j = c0 + e * T + tid;
              const CellFlags f = cell_update<MODE, V>(pca[e * T], pcb[e * T], psa[e * T], psb[e * T], rk,
                                                       j >= sh.i, j >= sh.id, j >= sh.s, j >= sh.su,
                                                       cn[e], sn[e]);
              emit_bp_stream<MODE>(bpc + e * (T / 32) * bp_words(MODE), f, pol);
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[slot]);  // this warp is done reading the slot
          V* qc = Cn + c0 + tid;
          V* qs = Sn + c0 + tid;
          if (geo.row_hint) {
#pragma unroll
            for (int e = 0; e < E; ++e) {
              st_hint(qc + e * T, cn[e], rpol);
              st_hint(qs + e * T, sn[e], rpol);
            }
          } else {
#pragma unroll
            for (int e = 0; e < E; ++e) {
              qc[e * T] = cn[e];
              qs[e * T] = sn[e];
            }
          }
          if (a.tab_c) {
            const int nc = ncol[i];
            const double g = a.info[inst[i]].scale;
#pragma unroll
            for (int e = 0; e < E; ++e) {
              const int j = c0 + e * T + tid;
              if (j < nc) {
                a.tab_c[(int64_t)(k + 1) * nc + j] = to_f64(cn[e], g);
                a.tab_s[(int64_t)(k + 1) * nc + j] = to_f64(sn[e], g);
              }
            }
          }
        }
        // publish row k+1 of this CTA's block of instance i
        named_barrier(1, T);
        if (tid == 0) {
          fence_acq_rel_cluster();
          fence_proxy_async_global();
          st_cluster_release(prog + i, (uint32_t)(k + 1));
        }
      }
    }
  }
  __syncthreads();
  cluster_barrier();  // no CTA leaves while others may still read its counters
  for (int i = 0; i < ni; ++i) {
    const int nc = ncol[i];
    if (tid == 0 && nc - 1 >= j0 && nc - 1 < j0 + B) {
      const double g = a.info[inst[i]].scale;
      a.info[inst[i]].end_c = to_f64(row(i, L[i] % NBUF, 0)[nc - 1], g);
      a.info[inst[i]].end_s = to_f64(row(i, L[i] % NBUF, 1)[nc - 1], g);
    }
  }
  __syncthreads();
  // the rows are dead: drop their L2 lines instead of writing them back
  for (int i = 0; i < ni; ++i)
    for (int buf = 0; buf < NBUF; ++buf)
      for (int rs = 0; rs < 2; ++rs)
        for (int x = tid * LINE; x < B; x += blockDim.x * LINE) discard_l2(row(i, buf, rs) + j0 + x);
}

// ---------------------------------------------------------------------------
// K2 own-block variant (int32 domain; EXPERIMENTAL, forced only with
// SPLITPLAN_DP_VARIANT=own): a cluster of G CTAs per instance, CTA q owning
// columns [q*B, (q+1)*B) of both rows in its own shared memory, updated in
// place top-down like the single-CTA kernel.  Only what other CTAs need goes
// through L2:
//  * a predecessor window (C or S row shifted by i, i+d, s or s+u) that lies
//    entirely in the own block is read straight from shared memory; windows
//    reaching left of the block are bulk-copied from the previous row's global
//    copy into per-window ring slots (full/empty mbarriers), and a window
//    straddling the block edge gets its own part patched into the slot;
//  * column p of the new row is stored to the global copy only if a CTA to
//    the right reads it next stage: p >= (q+1)*B - max(next stage's shifts).
// At cfg2 widths that removes ~3/4 of the window reads and ~1/3 of the row
// writes of the streaming kernel.  Ordering: the producer waits, per window,
// until the CTAs owning its remote columns published the previous row (RAW),
// and before the compute warps overwrite a global row buffer it checks that
// every CTA to the right has finished the stage that read it (WAR, NBUF
// buffers); a publisher warp releases the CTA's progress at cluster scope off
// the compute critical path, so stages pipeline as a wavefront.
// Measured on B200 (profiles/r01/own_experiment): 2.3e11 cells/s at cfg2
// against 4.7e11 for the streaming kernel, and 4.6e11 vs 1.0e12 for the
// single-CTA kernel at W = 1e4: the L2 traffic it saves is not what bounds
// the streaming kernel (removing every window copy there gains only 35 %),
// while its per-chunk bookkeeping doubles the instructions per cell and one
// CTA per SM halves the warps that hide the per-chunk barrier.  Kept with
// parity tests as a recorded experiment, not selected automatically.
struct OwnGeom {
  int G;        // CTAs per instance (cluster size)
  int NC;       // chunks per CTA
  int n_items;  // instances of the launch
  int pad;
};

__device__ __forceinline__ uint32_t ld_acquire_cta(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_addr(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta(uint32_t* p, uint32_t v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_addr(p)), "r"(v) : "memory");
}

// kind of a predecessor window [start, start + CH) for CTA q owning columns from j0:
// 0 = own (shared memory; for q == 0 also the NEG pad below column 0),
// 1 = remote (slot), 2 = straddles the block edge (remote part from the slot)
template <int CH>
__device__ __forceinline__ int own_win_kind(int q, int j0, int start) {
  if (q == 0 || start >= j0) return 0;
  return start + CH <= j0 ? 1 : 2;
}

template <int MODE, int T, int E, int NSW, int NBUF>
__global__ void __launch_bounds__(T + 64, (T <= 256 ? 2 : 1)) dp_own_kernel(DpArgs a, OwnGeom geo) {
  using V = typename VT<MODE>::T;
  constexpr int CH = T * E;
  constexpr int AL = 16 / (int)sizeof(V);
  constexpr int WIN = CH + AL;
  constexpr int PAD = stream_pad<V, CH>();
  constexpr int LINE = 128 / (int)sizeof(V);
  constexpr int NWARP = T / 32;
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);  // [NSW]
  uint64_t* empty = full + NSW;                         // [NSW]
  uint32_t* prog = reinterpret_cast<uint32_t*>(empty + NSW);  // stages published
  uint32_t* war = prog + 1;                                   // stages cleared for global stores
  uint32_t* done = prog + 2;                                  // stages finished by the compute warps

  const int G = geo.G, NC = geo.NC;
  const int B = NC * CH;
  const int q = (int)cluster_rank();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const DpWork wk = a.work[blockIdx.x / G];
  const int64_t inst = wk.inst;
  const int64_t lo = a.layer_off[inst];
  const int L = (int)(a.layer_off[inst + 1] - lo);
  const int ncol = (int)(a.info[inst].w_eff + 1);
  const bool sac = a.sac[inst] != 0;
  const int j0 = q * B;
  const int64_t span = (int64_t)PAD + (int64_t)G * B + LINE;
  V* const gbase = reinterpret_cast<V*>(a.rows + wk.row_off);  // [buf][C|S][PAD + G*B + LINE]
  auto grow = [&](int buf, int rs) { return gbase + (int64_t)(buf * 2 + rs) * span + PAD; };
  V* const ownC = reinterpret_cast<V*>(smem + 256) + CH;  // [CH pad | B own columns]
  V* const ownS = ownC + B + CH;
  V* const slots = ownS + B;  // [NSW][WIN]
  const V NEG = VT<MODE>::neg();
  const V ZERO = V(0);

  // row 0: own block in shared memory and in global buffer 0; NEG pads
  for (int x = tid - CH; x < B; x += blockDim.x) {
    const int j = j0 + x;
    const bool valid = x >= 0 && j < ncol;
    const V c = (valid && sac) ? ZERO : NEG, s = (valid && !sac) ? ZERO : NEG;
    ownC[x] = c;
    ownS[x] = s;
    if (x >= 0) {
      grow(0, 0)[j] = c;
      grow(0, 1)[j] = s;
    }
  }
  for (int buf = 0; buf < NBUF; ++buf) {
    if (q == 0)
      for (int x = tid - PAD; x < 0; x += blockDim.x) grow(buf, 0)[x] = grow(buf, 1)[x] = NEG;
    if (q == G - 1)
      for (int x = G * B + tid; x < G * B + LINE; x += blockDim.x) grow(buf, 0)[x] = grow(buf, 1)[x] = NEG;
  }
  if (tid == 0) {
    for (int b = 0; b < NSW; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], NWARP);
    }
    *prog = 0;
    *war = 0;
    *done = 0;
    fence_mbar_init();
  }
  fence_proxy_async_global();
  __threadfence();
  cluster_barrier();

  if (warp == NWARP) {
    // ---------------- producer warp: remote windows + WAR clearance ----------------
    const uint32_t peer = lane < G ? cluster_addr(smem_addr(prog), (uint32_t)lane) : 0u;
    uint32_t u = 0;
    StageShift sh = a.shifts[lo];
    for (int k = 0; k < L; ++k) {
      const StageShift shn = a.shifts[lo + min(k + 1, L - 1)];  // prefetch
      // WAR: the compute warps' stage-k stores go to buffer (k+1) % NBUF, last
      // read (stage k+1-NBUF) by the CTAs to the right
      const int war_need = k + 2 - NBUF;
      if (war_need > 0) {
        while (!__all_sync(0xffffffffu, lane <= q || lane >= G || ld_cluster_relaxed(peer) >= (uint32_t)war_need)) {
        }
        if (lane == 0) fence_acq_rel_cluster();
      }
      if (lane == 0) st_release_cta(war, (uint32_t)(k + 1));
      uint32_t ready = 0;  // lanes (CTAs) known to have published row k
      const V* Cr = grow(k % NBUF, 0);
      const V* Sr = grow(k % NBUF, 1);
      const int shf[4] = {sh.i, sh.id, sh.s, sh.su};
      for (int c = NC - 1; c >= 0; --c) {
        const int c0 = j0 + c * CH, ctop = c0 + CH;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const int start = c0 - min(shf[w], ctop);
          if (own_win_kind<CH>(q, j0, start) == 0) continue;
          // RAW: owners of the remote columns [max(start, 0), min(start + CH, j0))
          const int hi_col = min(start + CH, j0) - 1;
          const int olo = max(start, 0) / B;
          const int ohi = hi_col >= 0 ? hi_col / B : -1;
          const uint32_t want = (ohi >= olo) ? ((0xffffffffu >> (31 - ohi)) & (0xffffffffu << olo)) : 0u;
          if ((ready & want) != want) {
            do {
              ready = __ballot_sync(0xffffffffu, lane < G && ld_cluster_relaxed(peer) >= (uint32_t)k);
            } while ((ready & want) != want);
            if (lane == 0) {
              fence_acq_rel_cluster();
              fence_proxy_async_global();
            }
          }
          if (lane == 0) {
            // the window's columns left of the block (all of it unless it
            // straddles the edge; the compute warps fill in the own part)
            const int sa = start & ~(AL - 1);
            const uint32_t bytes = (uint32_t)(min(WIN, j0 - sa) * (int)sizeof(V));
            const int slot = (int)(u % NSW);
            mbar_wait(&empty[slot], ((u / NSW) & 1) ^ 1);
            mbar_expect_tx(&full[slot], bytes);
            const V* src = (w == 0 || w == 3) ? Cr : Sr;
            bulk_g2s(slots + slot * WIN, src + sa, bytes, &full[slot]);
          }
          ++u;
          __syncwarp();
        }
      }
      sh = shn;
    }
  } else if (warp == NWARP + 1) {
    // ---------------- publisher warp ----------------
    // publishes the latest stage the compute warps finished (their stores are
    // ordered before `done` by their stage-end barrier); the compute warps never
    // wait for it, and a slow release simply covers several stages at once
    if (lane == 0) {
      uint32_t pub = 0;
      while (pub < (uint32_t)L) {
        const uint32_t d = ld_acquire_cta(done);
        if (d == pub) {
          __nanosleep(64);
          continue;
        }
        fence_acq_rel_cluster();
        st_cluster_release(prog, d);
        pub = d;
      }
    }
    __syncwarp();
  } else {
    // ---------------- compute warps ----------------
    // Every predecessor read is an index into the shared array `sv` (so it is
    // an LDS): own rows at ownC / ownS, ring slots at slots.
    V* const sv = reinterpret_cast<V*>(smem);
    const int iC = (int)(ownC - sv), iS = (int)(ownS - sv), iSl = (int)(slots - sv);
    const uint64_t pol = evict_first_policy();
    uint32_t* const bpw = reinterpret_cast<uint32_t*>(a.bp + wk.bp_off) + warp * bp_words(MODE);
    const int64_t row_words = wk.bp_row_words;
    uint32_t u = 0;
    StageShift sh = a.shifts[lo];
    StageShift shn = a.shifts[lo + min(1, L - 1)];
    int64_t rbits = a.rv[lo];
    for (int k = 0; k < L; ++k) {
      const StageShift shn2 = a.shifts[lo + min(k + 2, L - 1)];  // prefetch
      const int64_t rbn = a.rv[lo + min(k + 1, L - 1)];
      const V rk = MODE == VM_INT32 ? (V)(int32_t)rbits : (V)__longlong_as_double(rbits);
      // global copy: only the columns a CTA to the right reads next stage
      int thrC = INT_MAX, thrS = INT_MAX;
      if (k + 1 < L && q + 1 < G) {
        thrC = j0 + B - max(shn.i, shn.su);
        thrS = j0 + B - max(shn.id, shn.s);
      }
      const int thr = min(thrC, thrS);
      V* const gC = grow((k + 1) % NBUF, 0);
      V* const gS = grow((k + 1) % NBUF, 1);
      uint32_t* const bprow = bpw + (int64_t)k * row_words;
      const int shf[4] = {sh.i, sh.id, sh.s, sh.su};
      const int rowi[4] = {iC - j0, iS - j0, iS - j0, iC - j0};  // own index of column p: rowi + p
      bool war_ok = false;
      for (int c = NC - 1; c >= 0; --c) {
        const int c0 = j0 + c * CH, ctop = c0 + CH;
        int base[4];
        uint32_t used = 0, strad = 0;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const int start = c0 - min(shf[w], ctop);
          base[w] = rowi[w] + start + tid;  // own-row index of this thread's first predecessor
          if (q > 0 && start < j0) {        // remote columns: this window has a ring slot
            const int slot = (int)(u % NSW);
            mbar_wait(&full[slot], (u / NSW) & 1);
            ++u;
            const int sa = start & ~(AL - 1);
            const int sb = iSl + slot * WIN - sa;  // slot index of column p: sb + p
            base[w] = sb + start + tid;
            used |= 1u << w;
            if (start + CH > j0) {  // straddles the block edge: copy the own part in
              strad = 1;
              const int ob = rowi[w];
              for (int p = j0 + tid; p < start + CH; p += T) sv[sb + p] = sv[ob + p];
            }
          }
        }
        if (strad) named_barrier(1, T);  // patched slots visible to every compute warp
        V cn[E], sn[E];
        uint32_t* const bpc = bprow + (c0 >> 5) * bp_words(MODE);
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int j = c0 + e * T + tid;
          const CellFlags f = cell_update<MODE, V>(sv[base[0] + e * T], sv[base[1] + e * T],
                                                   sv[base[2] + e * T], sv[base[3] + e * T], rk,
                                                   j >= sh.i, j >= sh.id, j >= sh.s, j >= sh.su, cn[e], sn[e]);
          emit_bp_stream<MODE>(bpc + e * (T / 32) * bp_words(MODE), f, pol);
        }
        // release this chunk's ring slots (the same slot sequence as above)
        __syncwarp();
        if (lane == 0) {
          uint32_t v = u;
#pragma unroll
          for (int w = 3; w >= 0; --w)
            if (used & (1u << w)) mbar_arrive(&empty[(int)(--v % NSW)]);
        }
        named_barrier(1, T);  // every read of this chunk's predecessors is done: update in place
        const int oi = iC + (c0 - j0) + tid, os = iS + (c0 - j0) + tid;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          sv[oi + e * T] = cn[e];
          sv[os + e * T] = sn[e];
        }
        if (ctop > thr) {
          if (!war_ok) {
            while (ld_acquire_cta(war) < (uint32_t)(k + 1)) {
            }
            war_ok = true;
          }
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int j = c0 + e * T + tid;
            if (j >= thrC) gC[j] = cn[e];
            if (j >= thrS) gS[j] = sn[e];
          }
        }
      }
      fence_proxy_async_global();  // the global row copy is read next by bulk copies
      named_barrier(1, T);         // stage done: own rows complete, global stores ordered
      if (tid == 0) st_release_cta(done, (uint32_t)(k + 1));
      sh = shn;
      shn = shn2;
      rbits = rbn;
    }
  }
  __syncthreads();
  cluster_barrier();  // no CTA leaves while others may still poll its counters
  if (tid == 0 && ncol - 1 >= j0 && ncol - 1 < j0 + B) {
    const double g = a.info[inst].scale;
    a.info[inst].end_c = to_f64(ownC[ncol - 1 - j0], g);
    a.info[inst].end_s = to_f64(ownS[ncol - 1 - j0], g);
  }
  // the global rows are dead: drop their L2 lines instead of writing them back
  for (int buf = 0; buf < NBUF; ++buf)
    for (int rs = 0; rs < 2; ++rs)
      for (int x = tid * LINE; x < B; x += blockDim.x * LINE) discard_l2(grow(buf, rs) + j0 + x);
}

// ---------------------------------------------------------------------------
// K2 grid variant: ONE very large instance (L = 1e5 stages x
// W = 1e7 columns) spread over every co-resident CTA of the GPU (cooperative
// launch).  Same producer-warp / bulk-copy / mbarrier-ring structure as the
// streaming kernel, but the per-CTA progress counters live in global memory
// and each producer waits only on the CTAs that own its windows: the owners
// of columns [j0 - max_shift - 16 B, j0 + B) for the rows it reads (RAW) and
// the CTAs that read its block two stages earlier (WAR on the triple-
// buffered rows).  With small per-stage shifts that is just the two
// neighbours, so the GPU runs as a wavefront with no grid-wide barrier.
// A launch advances a range of stages [k_begin, k_begin + k_count) from an
// initial row (the origin row or a checkpoint) and can write the final row
// (a checkpoint) and the range's back-pointers; the host chains launches
// into checkpoint / recompute passes when the full back-pointer table does
// not fit in memory.

constexpr int kMaxParts = 8;

// One huge instance over the whole GPU (or, partitioned, over several GPUs).
// The capacity axis can be split into `nparts` partitions of Gp CTAs each
// (one per device in a multi-GPU run): partition p owns global columns
// [p*Wp, (p+1)*Wp), Wp = Gp*B, keeps its own triple-buffered rows, and
// mirrors the left neighbour's last `halo` columns of every row in front of
// its column 0 -- the halo, written by the neighbour's CTAs with plain
// (peer) stores as they produce those columns.  Dependencies are computed
// in the global CTA index space, so the protocol is the same whether the
// partitions are launched together (one device, emulating several) or one
// per device.
struct GridArgs {
  const StageShift* shifts;  // stage records of the instance (index = stage)
  const int64_t* rv;         // stage values in the value domain
  const int2* reach;         // per stage: first reachable global column of the C / S row it reads
  int k_begin, k_count;      // stage range of this launch
  int ncol;                  // W_eff + 1
  int G, NC;                 // CTAs per partition, chunks per CTA
  int sac;
  const void* init_c;        // row k_begin, ncol values each, or null: origin row
  const void* init_s;
  void* out_c;               // row k_begin + k_count, or null
  void* out_s;
  uint32_t* bp;              // back-pointers of the range's stages, or null
  int64_t bp_row_words;
  uint32_t* progs[kMaxParts];  // per partition: [G] stages completed + 1 (zeroed)
  int nparts;                // partitions of the capacity axis
  int part_base;             // first partition of this launch
  int launch_parts;          // partitions of this launch (grid = launch_parts x G)
  int sys;                   // partitions on different devices: system-scope ordering
  int halo;                  // mirrored left-neighbour columns (multiple of 128 B)
  uint8_t* rows[kMaxParts];  // per partition: [3][C|S][NEG pad | halo | Wp | line]
};

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ int max_shift(const StageShift& sh) {
  return max(max(sh.i, sh.id), max(sh.s, sh.su));
}

template <int MODE, int T, int E, int NSLOT>
__global__ void __launch_bounds__(T + 32, 2) dp_grid_kernel(GridArgs a) {
  using V = typename VT<MODE>::T;
  constexpr int CH = T * E;
  constexpr int AL = 16 / (int)sizeof(V);
  constexpr int WIN = CH + AL;
  constexpr int PAD = stream_pad<V, CH>();  // NEG area in front of the halo
  constexpr int LINE = 128 / (int)sizeof(V);
  constexpr int NWARP = T / 32;
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + NSLOT;
  V* slots = reinterpret_cast<V*>(smem + 256);
  V* negwin = slots + NSLOT * 4 * WIN;  // [WIN] of NEG: windows below the reachable frontier

  const int G = a.G, NC = a.NC;
  const int part = a.part_base + (int)blockIdx.x / G;
  const int q = (int)blockIdx.x % G;
  const int GT = a.nparts * G;  // CTAs over the whole capacity axis
  const int gq = part * G + q;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int B = NC * CH;
  const int Wp = G * B;
  const int p0 = part * Wp;      // global column of this partition's local column 0
  const int j0 = q * B;          // local
  const int j0g = p0 + j0;       // global
  const int ncol = a.ncol;
  const int H = a.halo;
  const int64_t span = (int64_t)PAD + H + Wp + LINE;
  const V NEG = VT<MODE>::neg();
  const V ZERO = V(0);
  auto row_of = [&](int p, int buf, int rs) {
    return reinterpret_cast<V*>(a.rows[p]) + (int64_t)(buf * 2 + rs) * span + PAD + H;
  };
  auto row = [&](int buf, int rs) { return row_of(part, buf, rs); };
  auto owner = [&](int x) { return min(GT - 1, max(0, x) / B); };  // global CTA of global column x
  // progress counter of global CTA o (in its partition's -- possibly a peer device's -- memory)
  auto prog_of = [&](int o) { return a.progs[o / G] + (o % G); };
  auto publish = [&](uint32_t v) {
    if (a.sys) {
      __threadfence_system();
      fence_proxy_async_global();
      st_release_sys(prog_of(gq), v);
    } else {
      __threadfence();
      fence_proxy_async_global();
      st_release_gpu(prog_of(gq), v);
    }
  };
  const V* ic = reinterpret_cast<const V*>(a.init_c);
  const V* is = reinterpret_cast<const V*>(a.init_s);
  auto init_at = [&](int x, V& c, V& sv) {  // row k_begin at global column x
    const bool valid = x >= 0 && x < ncol;
    if (ic) {
      c = valid ? ic[x] : NEG;
      sv = valid ? is[x] : NEG;
    } else {
      c = (valid && a.sac) ? ZERO : NEG;
      sv = (valid && !a.sac) ? ZERO : NEG;
    }
  };

  for (int buf = 0; buf < kRowBufs; ++buf) {
    V* Cb = row(buf, 0);
    V* Sb = row(buf, 1);
    if (q == 0) {
      for (int x = tid - PAD - H; x < -H; x += blockDim.x) Cb[x] = Sb[x] = NEG;  // NEG area
      // halo of buffer 0: row k_begin of the neighbour's last columns (all NEG
      // in partition 0).  Buffers 1 and 2 belong to the neighbour's CTAs, which
      // write them before any read (RAW) -- never touch them here.
      if (buf == 0)
        for (int x = tid - H; x < 0; x += blockDim.x) {
          V c = NEG, sv = NEG;
          if (part > 0) init_at(p0 + x, c, sv);
          Cb[x] = c;
          Sb[x] = sv;
        }
      else if (part == 0)
        for (int x = tid - H; x < 0; x += blockDim.x) Cb[x] = Sb[x] = NEG;
    }
    if (q == G - 1)
      for (int x = Wp + tid; x < Wp + LINE; x += blockDim.x) Cb[x] = Sb[x] = NEG;
    if (buf == 0)
      for (int j = j0 + tid; j < j0 + B; j += blockDim.x) init_at(p0 + j, Cb[j], Sb[j]);
  }
  for (int x = tid; x < WIN; x += blockDim.x) negwin[x] = NEG;
  if (tid == 0) {
    for (int b = 0; b < NSLOT; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], NWARP);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) publish(1u);  // rows initialised (counter = completed stages + 1)

  if (warp == NWARP) {
    // ---------------- producer warp ----------------
    uint32_t u = 0;
    for (int t = 0; t < a.k_count; ++t) {
      const int k = a.k_begin + t;
      const StageShift sh = a.shifts[k];
      // RAW: owners of the windows read this stage (row t complete => counter >= t + 1)
      const int lo_o = owner(j0g - max_shift(sh) - AL);
      // WAR: CTAs that read this block's target buffers (own rows and the
      // right neighbour's halo copy) two stages ago
      int hi_o = gq;
      if (t >= 2) hi_o = owner(j0g + B - 1 + max_shift(a.shifts[k - 2]) + CH + AL);
      for (int o0 = lo_o; o0 <= hi_o; o0 += 32) {
        const int o = o0 + lane;
        const uint32_t need = o <= gq ? (uint32_t)(t + 1) : (uint32_t)max(t - 1, 0) + 1u;
        // (a watchdog turns a lost partition -- e.g. launches that were not
        // co-scheduled -- into a launch failure instead of a hang)
        const long long t0 = clock64();
        for (uint32_t it = 1;; ++it) {
          const bool ok = o > hi_o || (a.sys ? ld_acquire_sys(prog_of(o)) : ld_acquire_gpu(prog_of(o))) >= need;
          if (__all_sync(0xffffffffu, ok)) break;
          if ((it & 1023u) == 0 && clock64() - t0 > (30ll << 30)) __trap();
        }
      }
      if (lane == 0) {
        fence_proxy_async_global();
        const V* Cc = row(t % kRowBufs, 0);
        const V* Sc = row(t % kRowBufs, 1);
        const V* src[4] = {Cc, Sc, Sc, Cc};
        const int shf[4] = {sh.i, sh.id, sh.s, sh.su};
        const int2 rch = a.reach ? a.reach[a.k_begin + t] : make_int2(0, 0);
        const int mrow[4] = {rch.x, rch.y, rch.y, rch.x};
        for (int c = 0; c < NC; ++c, ++u) {
          const int slot = (int)(u % NSLOT);
          mbar_wait(&empty[slot], ((u / NSLOT) & 1) ^ 1);
          const int c0g = j0g + c * CH, ctop = c0g + CH;
          uint32_t ncopy = 0;
#pragma unroll
          for (int w = 0; w < 4; ++w) ncopy += c0g - min(shf[w], ctop) + CH > mrow[w] ? 1u : 0u;
          mbar_expect_tx(&full[slot], ncopy * WIN * sizeof(V));
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            const int start = c0g - min(shf[w], ctop);
            if (start + CH <= mrow[w]) continue;  // below the reachable frontier: all NEG, no copy
            // Partition 0 keeps NEG in front of column 0 (halo + NEG area), so
            // partially negative windows read it in place.  In later
            // partitions start < 0 only when the shift was clamped (every cell
            // of the window unreachable): read the NEG area.
            const int local = (start < 0 && part > 0) ? -H - PAD : (start & ~(AL - 1)) - p0;
            bulk_g2s(slots + (slot * 4 + w) * WIN, src[w] + local, WIN * sizeof(V), &full[slot]);
          }
        }
      }
      __syncwarp();
    }
  } else {
    // ---------------- compute warps ----------------
    const uint64_t pol = evict_first_policy();
    uint32_t u = 0;
    StageShift sh_next = a.shifts[a.k_begin];
    int64_t rbits_next = a.rv[a.k_begin];
    // global columns mirrored into the right neighbour's halo
    const int halo_lo = part + 1 < a.nparts ? p0 + Wp - H : INT_MAX;
    for (int t = 0; t < a.k_count; ++t) {
      const StageShift sh = sh_next;
      const int64_t rbits = rbits_next;
      if (t + 1 < a.k_count) {
        sh_next = a.shifts[a.k_begin + t + 1];
        rbits_next = a.rv[a.k_begin + t + 1];
      }
      const V rk = MODE == VM_INT32 ? (V)(int32_t)rbits : (V)__longlong_as_double(rbits);
      V* Cn = row((t + 1) % kRowBufs, 0);
      V* Sn = row((t + 1) % kRowBufs, 1);
      uint32_t* bprow = a.bp ? a.bp + (int64_t)t * a.bp_row_words + warp * bp_words(MODE) : nullptr;
      const int2 rch = a.reach ? a.reach[a.k_begin + t] : make_int2(0, 0);
      // every cell of row t+1 below both frontiers is unreachable
      const int64_t next_front = a.reach ? min(min((int64_t)rch.x + sh.i, (int64_t)rch.y + sh.id),
                                               min((int64_t)rch.y + sh.s, (int64_t)rch.x + sh.su))
                                         : 0;
      for (int c = 0; c < NC; ++c, ++u) {
        const int slot = (int)(u % NSLOT);
        const int c0 = j0 + c * CH;       // local
        const int c0g = p0 + c0, ctop = c0g + CH;
        const int sa = c0g - min(sh.i, ctop), sb = c0g - min(sh.id, ctop);
        const int sc = c0g - min(sh.s, ctop), sd = c0g - min(sh.su, ctop);
        const V* ws = slots + slot * 4 * WIN + tid;
        const V* pca = (sa + CH > rch.x ? ws + 0 * WIN : negwin + tid) + (sa & (AL - 1));
        const V* pcb = (sb + CH > rch.y ? ws + 1 * WIN : negwin + tid) + (sb & (AL - 1));
        const V* psa = (sc + CH > rch.y ? ws + 2 * WIN : negwin + tid) + (sc & (AL - 1));
        const V* psb = (sd + CH > rch.x ? ws + 3 * WIN : negwin + tid) + (sd & (AL - 1));
        mbar_wait(&full[slot], (u / NSLOT) & 1);
        V cn[E], sn[E];
        CellFlags f[E];
        const bool dead = (int64_t)ctop <= next_front;  // whole chunk unreachable: NEG, no back-pointers
        if (dead) {
#pragma unroll
          for (int e = 0; e < E; ++e) cn[e] = sn[e] = NEG;
        } else {
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int j = c0g + e * T + tid;
            f[e] = cell_update<MODE, V>(pca[e * T], pcb[e * T], psa[e * T], psb[e * T], rk, j >= sh.i,
                                        j >= sh.id, j >= sh.s, j >= sh.su, cn[e], sn[e]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        if (bprow && !dead) {
          uint32_t* bpc = bprow + (c0g >> 5) * bp_words(MODE);
#pragma unroll
          for (int e = 0; e < E; ++e) emit_bp_stream<MODE>(bpc + e * (T / 32) * bp_words(MODE), f[e], pol);
        }
        V* qc = Cn + c0 + tid;
        V* qs = Sn + c0 + tid;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          qc[e * T] = cn[e];
          qs[e * T] = sn[e];
        }
        if (ctop > halo_lo) {  // the right neighbour mirrors these columns
          V* hc = row_of(part + 1, (t + 1) % kRowBufs, 0) - (p0 + Wp);
          V* hs = row_of(part + 1, (t + 1) % kRowBufs, 1) - (p0 + Wp);
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int j = c0g + e * T + tid;
            if (j >= halo_lo) {
              hc[j] = cn[e];
              hs[j] = sn[e];
            }
          }
        }
      }
      named_barrier(1, T);
      if (tid == 0) publish((uint32_t)(t + 2));
    }
    // the range's final row (this CTA's own block: its own writes)
    if (a.out_c) {
      named_barrier(1, T);
      V* oc = reinterpret_cast<V*>(a.out_c);
      V* os = reinterpret_cast<V*>(a.out_s);
      const V* Cf = row(a.k_count % kRowBufs, 0);
      const V* Sf = row(a.k_count % kRowBufs, 1);
      for (int j = j0 + tid; j < j0 + B && p0 + j < ncol; j += T) {
        oc[p0 + j] = Cf[j];
        os[p0 + j] = Sf[j];
      }
    }
  }
}

// End of the forward pass of a grid-solved instance: the end side from the
// final row's last cell (planner.py:190-200), or the infeasible policy.
// state = {j, client side, infeasible}.
// ---------------------------------------------------------------------------
// K2 grid variant with ONE row buffer (single partition, every stage's
// shifts <= the halo width): the rows of a 1e7-column instance are 80 MB
// instead of 240 MB with three buffers, so they stay in L2 instead of
// streaming through HBM (profiles/r01/dp_grid_ncu_summary.json: 15.5 B/cell
// of DRAM traffic with three buffers).  Each CTA updates its block IN PLACE,
// chunks top-down: every predecessor window of chunk c lies below the top of
// chunk c (reads go left), so the chunks above c that already hold the new
// row are never read again this stage, and window copies already sit in
// shared-memory slots before chunk c stores over them.  Nobody else reads the
// main buffer: the right neighbour takes this block's last `hw` columns from
// a small per-CTA halo buffer (3 stage slots) written alongside the row.
// Producer waits per stage: own and left neighbour finished the previous
// stage (RAW), right neighbour finished the stage two back (WAR on the halo
// slot this stage overwrites).
struct GridInplaceArgs {
  const StageShift* shifts;
  const int64_t* rv;
  const int2* reach;
  int k_begin, k_count;
  int ncol, G, NC, sac, hw;  // hw: halo columns (multiple of 128 B, <= B)
  const void* init_c;
  const void* init_s;
  void* out_c;
  void* out_s;
  uint32_t* bp;
  int64_t bp_row_words;
  uint32_t* prog;  // [G] completed stages + 1 (zeroed)
  uint8_t* rows;   // [C|S][PAD | G*B | line]
  uint8_t* halo;   // [G][3][C|S][hw]
  int row_hint;    // 1: row stores with an L2 evict_last policy (SPLITPLAN_ROW_EVICT_LAST)
};

template <int MODE, int T, int E, int NSLOT>
__global__ void __launch_bounds__(T + 32, 2) dp_grid_inplace_kernel(GridInplaceArgs a) {
  using V = typename VT<MODE>::T;
  constexpr int CH = T * E;
  constexpr int AL = 16 / (int)sizeof(V);
  constexpr int WIN = CH + AL;
  constexpr int PAD = stream_pad<V, CH>();
  constexpr int LINE = 128 / (int)sizeof(V);
  constexpr int NWARP = T / 32;
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + NSLOT;
  V* slots = reinterpret_cast<V*>(smem + 256);
  V* negwin = slots + NSLOT * 4 * WIN;  // [WIN] of NEG: windows below the reachable frontier

  const int G = a.G, NC = a.NC;
  const int q = (int)blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int B = NC * CH;
  const int Wt = G * B;
  const int j0 = q * B;
  const int ncol = a.ncol, hw = a.hw;
  const int64_t span = (int64_t)PAD + Wt + LINE;
  const V NEG = VT<MODE>::neg();
  const V ZERO = V(0);
  V* const Cm = reinterpret_cast<V*>(a.rows) + PAD;          // C row, column 0
  V* const Sm = reinterpret_cast<V*>(a.rows) + span + PAD;   // S row, column 0
  // halo of CTA o, stage slot t % 3: columns [o*B + B - hw, o*B + B) of row t
  auto halo = [&](int o, int slot, int rs) {
    return reinterpret_cast<V*>(a.halo) + ((int64_t)(o * 3 + slot) * 2 + rs) * hw;
  };
  const V* ic = reinterpret_cast<const V*>(a.init_c);
  const V* is = reinterpret_cast<const V*>(a.init_s);

  // row k_begin in the main buffer, its top hw columns in halo slot 0, NEG pads
  for (int x = j0 + tid; x < j0 + B; x += blockDim.x) {
    const bool valid = x < ncol;
    V c, s;
    if (ic) {
      c = valid ? ic[x] : NEG;
      s = valid ? is[x] : NEG;
    } else {
      c = (valid && a.sac) ? ZERO : NEG;
      s = (valid && !a.sac) ? ZERO : NEG;
    }
    Cm[x] = c;
    Sm[x] = s;
    if (x >= j0 + B - hw) {
      halo(q, 0, 0)[x - (j0 + B - hw)] = c;
      halo(q, 0, 1)[x - (j0 + B - hw)] = s;
    }
  }
  if (q == 0)
    for (int x = tid - PAD; x < 0; x += blockDim.x) Cm[x] = Sm[x] = NEG;
  if (q == G - 1)
    for (int x = Wt + tid; x < Wt + LINE; x += blockDim.x) Cm[x] = Sm[x] = NEG;
  for (int x = tid; x < WIN; x += blockDim.x) negwin[x] = NEG;
  if (tid == 0) {
    for (int b = 0; b < NSLOT; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], NWARP);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    fence_proxy_async_global();
    st_release_gpu(&a.prog[q], 1u);
  }

  if (warp == NWARP) {
    // ---------------- producer warp ----------------
    uint32_t u = 0;
    for (int t = 0; t < a.k_count; ++t) {
      const StageShift sh = a.shifts[a.k_begin + t];
      // lane 0: own block (row t complete), lane 1: left neighbour (its halo
      // of row t), lane 2: right neighbour (finished stage t - 2: halo slot reuse)
      const int o = lane == 0 ? q : (lane == 1 ? q - 1 : q + 1);
      const bool watch = lane < 3 && o >= 0 && o < G;
      const uint32_t need = lane < 2 ? (uint32_t)(t + 1) : (uint32_t)max(t - 1, 0) + 1u;
      const long long t0 = clock64();
      for (uint32_t it = 1;; ++it) {
        if (__all_sync(0xffffffffu, !watch || ld_acquire_gpu(&a.prog[o]) >= need)) break;
        if ((it & 1023u) == 0 && clock64() - t0 > (30ll << 30)) __trap();
      }
      if (lane == 0) {
        fence_proxy_async_global();
        const V* hc = q > 0 ? halo(q - 1, t % 3, 0) - (j0 - hw) : nullptr;  // index by global column
        const V* hs = q > 0 ? halo(q - 1, t % 3, 1) - (j0 - hw) : nullptr;
        const int shf[4] = {sh.i, sh.id, sh.s, sh.su};
        const int2 rch = a.reach ? a.reach[a.k_begin + t] : make_int2(0, 0);
        const int mrow[4] = {rch.x, rch.y, rch.y, rch.x};
        for (int c = NC - 1; c >= 0; --c, ++u) {
          const int slot = (int)(u % NSLOT);
          mbar_wait(&empty[slot], ((u / NSLOT) & 1) ^ 1);
          const int c0 = j0 + c * CH, ctop = c0 + CH;
          uint32_t ncopy = 0;
#pragma unroll
          for (int w = 0; w < 4; ++w) ncopy += c0 - min(shf[w], ctop) + CH > mrow[w] ? 1u : 0u;
          mbar_expect_tx(&full[slot], ncopy * WIN * sizeof(V));
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            const bool cw = w == 0 || w == 3;
            const int start = c0 - min(shf[w], ctop);
            if (start + CH <= mrow[w]) continue;  // below the reachable frontier: all NEG, no copy
            V* dst = slots + (slot * 4 + w) * WIN;
            if (q == 0 || start < 0) {  // partition start: NEG pad in front of column 0
              const int sa = start < 0 && q > 0 ? -PAD : (start & ~(AL - 1));
              bulk_g2s(dst, (cw ? Cm : Sm) + sa, WIN * sizeof(V), &full[slot]);
              continue;
            }
            const int sa = start & ~(AL - 1);
            const int split = min(max(j0 - sa, 0), WIN);  // values from the left halo
            if (split > 0)
              bulk_g2s(dst, (cw ? hc : hs) + sa, split * sizeof(V), &full[slot]);
            if (split < WIN)
              bulk_g2s(dst + split, (cw ? Cm : Sm) + sa + split, (WIN - split) * sizeof(V), &full[slot]);
          }
        }
      }
      __syncwarp();
    }
  } else {
    // ---------------- compute warps ----------------
    const uint64_t pol = evict_first_policy();
    const uint64_t rpol = evict_last_policy();
    uint32_t u = 0;
    StageShift sh_next = a.shifts[a.k_begin];
    int64_t rbits_next = a.rv[a.k_begin];
    const int hlo = j0 + B - hw;  // first column mirrored into this CTA's halo
    for (int t = 0; t < a.k_count; ++t) {
      const StageShift sh = sh_next;
      const int64_t rbits = rbits_next;
      if (t + 1 < a.k_count) {
        sh_next = a.shifts[a.k_begin + t + 1];
        rbits_next = a.rv[a.k_begin + t + 1];
      }
      const V rk = MODE == VM_INT32 ? (V)(int32_t)rbits : (V)__longlong_as_double(rbits);
      V* const hc = halo(q, (t + 1) % 3, 0) - hlo;
      V* const hs = halo(q, (t + 1) % 3, 1) - hlo;
      uint32_t* bprow = a.bp ? a.bp + (int64_t)t * a.bp_row_words + warp * bp_words(MODE) : nullptr;
      const int2 rch = a.reach ? a.reach[a.k_begin + t] : make_int2(0, 0);
      const int64_t next_front = a.reach ? min(min((int64_t)rch.x + sh.i, (int64_t)rch.y + sh.id),
                                               min((int64_t)rch.y + sh.s, (int64_t)rch.x + sh.su))
                                         : 0;
      for (int c = NC - 1; c >= 0; --c, ++u) {
        const int slot = (int)(u % NSLOT);
        const int c0 = j0 + c * CH, ctop = c0 + CH;
        const int sa = c0 - min(sh.i, ctop), sb = c0 - min(sh.id, ctop);
        const int sc = c0 - min(sh.s, ctop), sd = c0 - min(sh.su, ctop);
        const V* ws = slots + slot * 4 * WIN + tid;
        const V* pca = (sa + CH > rch.x ? ws + 0 * WIN : negwin + tid) + (sa & (AL - 1));
        const V* pcb = (sb + CH > rch.y ? ws + 1 * WIN : negwin + tid) + (sb & (AL - 1));
        const V* psa = (sc + CH > rch.y ? ws + 2 * WIN : negwin + tid) + (sc & (AL - 1));
        const V* psb = (sd + CH > rch.x ? ws + 3 * WIN : negwin + tid) + (sd & (AL - 1));
        mbar_wait(&full[slot], (u / NSLOT) & 1);
        V cn[E], sn[E];
        CellFlags f[E];
        const bool dead = (int64_t)ctop <= next_front;  // whole chunk unreachable: NEG, no back-pointers
        if (dead) {
#pragma unroll
          for (int e = 0; e < E; ++e) cn[e] = sn[e] = NEG;
        } else {
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int j = c0 + e * T + tid;
            f[e] = cell_update<MODE, V>(pca[e * T], pcb[e * T], psa[e * T], psb[e * T], rk, j >= sh.i,
                                        j >= sh.id, j >= sh.s, j >= sh.su, cn[e], sn[e]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        if (bprow && !dead) {
          uint32_t* bpc = bprow + (c0 >> 5) * bp_words(MODE);
#pragma unroll
          for (int e = 0; e < E; ++e) emit_bp_stream<MODE>(bpc + e * (T / 32) * bp_words(MODE), f[e], pol);
        }
        V* qc = Cm + c0 + tid;
        V* qs = Sm + c0 + tid;
        if (a.row_hint) {  // keep the rows ahead of the streamed back-pointers in L2
#pragma unroll
          for (int e = 0; e < E; ++e) {
            st_hint(qc + e * T, cn[e], rpol);
            st_hint(qs + e * T, sn[e], rpol);
          }
        } else {
#pragma unroll
          for (int e = 0; e < E; ++e) {
            qc[e * T] = cn[e];
            qs[e * T] = sn[e];
          }
        }
        if (ctop > hlo) {
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int j = c0 + e * T + tid;
            if (j >= hlo) {
              hc[j] = cn[e];
              hs[j] = sn[e];
            }
          }
        }
      }
      named_barrier(1, T);
      if (tid == 0) {
        __threadfence();
        fence_proxy_async_global();
        st_release_gpu(&a.prog[q], (uint32_t)(t + 2));
      }
    }
    if (a.out_c) {
      named_barrier(1, T);
      V* oc = reinterpret_cast<V*>(a.out_c);
      V* os = reinterpret_cast<V*>(a.out_s);
      for (int j = j0 + tid; j < j0 + B && j < ncol; j += T) {
        oc[j] = Cm[j];
        os[j] = Sm[j];
      }
    }
  }
}

__global__ void grid_end_kernel(sp_instances in, InstInfo* info, int64_t inst, const void* last_c,
                                const void* last_s, int64_t* state) {
  const InstInfo inf = info[inst];
  const int64_t jl = inf.w_eff;
  double ec, es;
  if (inf.mode == VM_INT32) {
    ec = to_f64(reinterpret_cast<const int32_t*>(last_c)[jl], inf.scale);
    es = to_f64(reinterpret_cast<const int32_t*>(last_s)[jl], inf.scale);
  } else {
    ec = reinterpret_cast<const double*>(last_c)[jl];
    es = reinterpret_cast<const double*>(last_s)[jl];
  }
  info[inst].end_c = ec;
  info[inst].end_s = es;
  const int8_t must = in.must_end_at ? in.must_end_at[inst] : (int8_t)-1;
  if (must == 1) es = -INFINITY;
  else if (must == 0) ec = -INFINITY;
  const double pmax = (es > ec) ? es : ec;
  state[0] = jl;
  state[1] = ec >= es ? 1 : 0;
  state[2] = pmax == -INFINITY ? 1 : 0;
}

// Walk one segment of back-pointers (stages k_begin + k_count - 1 .. k_begin)
// from state {j, side}, writing pi; the same decisions as backtrack_kernel.
__global__ void grid_backtrack_kernel(sp_instances in, int64_t inst, const StageShift* shifts,
                                      const uint32_t* bp, int64_t row_words, int mode, int k_begin,
                                      int k_count, int64_t* state, sp_policies out) {
  const int64_t lo = in.layer_off[inst];
  int64_t j = state[0];
  bool client = state[1] != 0;
  const int nw = bp_words(mode);
  uint8_t* pi = out.pi + lo;
  for (int t = k_count - 1; t >= 0; --t) {
    const int k = k_begin + t;
    const uint32_t* grp = bp + (int64_t)t * row_words + (j >> 5) * nw;
    const uint32_t bit = 1u << (j & 31);
    const bool c_stay = grp[0] & bit, s_stay = grp[1] & bit;
    const bool c_sw = nw == 4 ? (grp[2] & bit) != 0 : !c_stay;
    const bool s_sw = nw == 4 ? (grp[3] & bit) != 0 : !s_stay;
    const StageShift sh = shifts[lo + k];
    if (client) {
      pi[k] = 1;
      if (c_stay) {
        j -= sh.i;
      } else if (c_sw) {
        j -= sh.id;
        client = false;
      } else {
        out.status[inst] = SP_ERR_BACKTRACE;
        state[2] = 2;
        return;
      }
    } else {
      pi[k] = 0;
      if (s_stay) {
        j -= sh.s;
      } else if (s_sw) {
        j -= sh.su;
        client = true;
      } else {
        out.status[inst] = SP_ERR_BACKTRACE;
        state[2] = 2;
        return;
      }
    }
  }
  state[0] = j;
  state[1] = client ? 1 : 0;
}

// ---------------------------------------------------------------------------
// _finish (planner.py:88-101) for a placement already written to pi

__device__ void finish_policy(const sp_instances& in, int64_t inst, int64_t lo, int L,
                              int32_t* idx, sp_policies& out, bool feasible_hint, bool hint_value) {
  const uint8_t* pi = out.pi + lo;
  const bool sac = in.source_at_client[inst] != 0;
  int64_t lat = 0;
  int prev = sac ? 1 : 0;
  int n1 = 0;
  for (int k = 0; k < L; ++k) {
    const int x = pi[k];
    if (x) {
      lat += in.client_units[lo + k] + (prev == 0 ? in.down_units[lo + k] : 0);
      ++n1;
    } else {
      lat += in.server_units[lo + k] + (prev == 1 ? in.up_units[lo + k] : 0);
    }
    prev = x;
  }
  int a = 0, b = n1;
  for (int k = 0; k < L; ++k) {
    if (pi[k]) idx[a++] = k;
    else idx[b++] = k;
  }
  const double* r = in.r + lo;
  const double cv = np_sum([&](int64_t m) { return r[idx[m]]; }, n1);
  const double sl = np_sum([&](int64_t m) { return r[idx[n1 + m]]; }, L - n1);
  out.client_value[inst] = cv;
  out.server_load[inst] = sl;
  out.integer_latency[inst] = lat;
  out.feasible[inst] = feasible_hint ? (hint_value ? 1 : 0) : (lat <= in.budget[inst] ? 1 : 0);
}


// _finish of one grid-solved instance; state[2]: 0 ok, 1 infeasible, 2 backtrace error
__global__ void grid_finish_kernel(sp_instances in, int64_t inst, const int64_t* state,
                                   int32_t* idx_scratch, sp_policies out) {
  const int64_t lo = in.layer_off[inst];
  const int L = (int)(in.layer_off[inst + 1] - lo);
  if (state[2] == 2) return;  // status already set
  if (state[2] == 1)
    for (int k = 0; k < L; ++k) out.pi[lo + k] = 0;
  finish_policy(in, inst, lo, L, idx_scratch + lo, out, state[2] == 1, false);
  out.status[inst] = SP_OK;
}

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
// bulk-copy ring depth of the grid kernel (T = 256, E = 4)
template <int MODE> constexpr int ring_slots() { return MODE == VM_INT32 ? 6 : 3; }
inline int ring_slots_rt(int mode) { return mode == VM_INT32 ? 6 : 3; }
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

constexpr int kGridT = 256, kGridE = 4;
constexpr int kGridCH = kGridT * kGridE;
constexpr int64_t kGridMinCols = (int64_t)1 << 22;
enum { DPV_GRID = 5 };

size_t grid_smem(int mode) {
  const size_t vb = value_bytes(mode);  // ring slots + one NEG window
  return 256 + (size_t)(ring_slots_rt(mode) * 4 + 1) * (kGridCH + 16 / vb) * vb;
}

template <int MODE>
int grid_resident() {
  auto kern = dp_grid_kernel<MODE, kGridT, kGridE, ring_slots<MODE>()>;
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
  auto kern = dp_grid_kernel<MODE, kGridT, kGridE, ring_slots<MODE>()>;
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
  auto kern = dp_grid_inplace_kernel<MODE, kGridT, kGridE, ring_slots<MODE>()>;
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
  const int64_t nchunks = (ncol + kGridCH - 1) / kGridCH;
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
  const int64_t B = (int64_t)NC * kGridCH;
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
  const int64_t span = (kGridCH + line) + halo + G * B + line;
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
           size_t ws_bytes, cudaStream_t st) {
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
