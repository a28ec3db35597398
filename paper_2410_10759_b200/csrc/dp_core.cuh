// Value domains, the prep kernel (W_eff, value domain, clamped stage shifts,
// reachable frontiers), the per-cell DP update and back-pointer packing shared by
// every K2 variant, and the single-CTA kernel dp_stage_kernel.
//
// Fragment of sp_planner.cu: included there inside namespace sp::(anonymous),
// after the declarations it uses; not a standalone header.
#pragma once

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

// binary (Stein) gcd: shifts and subtractions, no 64-bit division
// exact remainder of integral doubles 0 <= v, 0 < d < 2^53: q = floor(v / d)
// may be one off, v - q*d is an integer below 2d in magnitude and the fma
// computes it exactly; one correction step fixes q
__device__ __forceinline__ double rem_exact(double v, double d) {
  const double q = floor(__ddiv_rn(v, d));
  double r = __fma_rn(-q, d, v);
  if (r < 0.0) r = __dadd_rn(r, d);
  else if (r >= d) r = __dadd_rn(r, -d);
  return r;
}
__device__ __forceinline__ double gcd_f64(double a, double b) {
  while (b != 0.0) {
    const double t = rem_exact(a, b);
    a = b;
    b = t;
  }
  return a;
}

__device__ __forceinline__ uint64_t gcd_u64(uint64_t a, uint64_t b) {
  if (a == 0) return b;
  if (b == 0) return a;
  const int shift = __ffsll((long long)(a | b)) - 1;
  a >>= __ffsll((long long)a) - 1;
  do {
    b >>= __ffsll((long long)b) - 1;
    if (a > b) {
      const uint64_t t = a;
      a = b;
      b = t;
    }
    b -= a;
  } while (b);
  return a << shift;
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

// One warp per instance (four per 128-thread block), no block barriers.
// flag (optional): set to 1 for every instance (the breakpoint-list tier
// clears it for the instances it solves).  steps_hi > 0: instances the
// breakpoint-list tier takes (not NaN, steps_lo[domain] <= W_eff + 1 <
// steps_hi) get the trivial frontier (0, 0) instead of the sequential
// recurrence -- only the dense kernels use it, and skipping nothing is exact.
constexpr int kPrepWarps = 4;
__global__ void __launch_bounds__(32 * kPrepWarps) prep_kernel(sp_instances in, InstInfo* info, StageShift* shifts,
                                                               int64_t* rv, int2* reach, int32_t* flag,
                                                               int64_t steps_hi = 0, int64_t steps_lo_i32 = 0,
                                                               int64_t steps_lo_f64 = 0) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * kPrepWarps;
  for (int64_t k = (int64_t)blockIdx.x * kPrepWarps + (threadIdx.x >> 5); k < in.n; k += nw) {
    const int64_t lo = in.layer_off[k], hi = in.layer_off[k + 1];
    int64_t worst = 0;
    int finite = 1, integral = 1;
    uint64_t isum = 0, orv = 0;
    for (int64_t l = lo + lane; l < hi; l += 32) {
      worst += max(in.client_units[l] + in.down_units[l], in.server_units[l] + in.up_units[l]);
      const double r = in.r[l];
      if (!isfinite(r)) {
        finite = 0;
      } else if (r != floor(r) || r >= 9007199254740992.0) {
        integral = 0;
      } else {
        const uint64_t v = (uint64_t)r;  // r >= 0 (problem.py:151-153)
        isum = min(isum + v, (uint64_t)1 << 62);
        orv |= v;
      }
    }
    {
      const uint64_t sat = (uint64_t)1 << 62;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        worst += __shfl_xor_sync(0xffffffffu, worst, o);
        finite &= __shfl_xor_sync(0xffffffffu, finite, o);
        integral &= __shfl_xor_sync(0xffffffffu, integral, o);
        isum = min(isum + __shfl_xor_sync(0xffffffffu, isum, o), sat);
        orv |= __shfl_xor_sync(0xffffffffu, orv, o);
      }
    }
    // The int32 domain stores r / g for any common divisor g (the values are
    // g * v exactly either way); the largest power of two dividing every r
    // (the lowest set bit of their OR) usually leaves the sums in range
    // (model FLOP counts carry large powers of two), and only when it does
    // not is the exact gcd computed -- a second pass of binary gcds.
    uint64_t g = orv ? (orv & (~orv + 1)) : 1;
    if (finite && integral && isum < ((uint64_t)1 << 53) && isum / g > (uint64_t)INT32_MAX) {
      // Euclid on exact doubles (every r < 2^53): once the running gcd has
      // settled, each further r costs one exact remainder
      double gg = 0.0;
      for (int64_t l = lo + lane; l < hi; l += 32) gg = gcd_f64(gg, in.r[l]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) gg = gcd_f64(gg, __shfl_xor_sync(0xffffffffu, gg, o));
      g = gg > 0.0 ? (uint64_t)gg : 1;
    }
    const int64_t W = min(in.budget[k], worst);
    int32_t mode;
    if (!finite) mode = VM_F64_NAN;
    else if (integral && isum < ((uint64_t)1 << 53) && isum / g <= (uint64_t)INT32_MAX) mode = VM_INT32;
    else mode = VM_F64;
    if (lane == 0) {
      InstInfo r;
      r.w_eff = W;
      r.scale = (double)g;
      r.end_c = -INFINITY;
      r.end_s = -INFINITY;
      r.mode = mode;
      r.pad = 0;
      info[k] = r;
      if (flag) flag[k] = 1;
    }
    const int64_t cap = min(W + 1, kMaxCols);
    // reachable frontier: the first column of row k of C and of S that holds a
    // reachable value (rows are monotone in j; every column below it is
    // unreachable, NEG-like).  reach[lo + k] describes the row stage k reads.
    // Not in the NaN domain, where "unreachable" cells may hold NaN.  The
    // recurrence is sequential: every lane runs it over the warp's 32 stage
    // records (shuffled in turn) and keeps the value of its own stage.
    const bool sac = in.source_at_client[k] != 0;
    int64_t mc = sac ? 0 : cap, ms = sac ? cap : 0;
    const bool trivial = mode == VM_F64_NAN ||
                         (steps_hi > 0 && W + 1 < steps_hi && W + 1 >= (mode == VM_INT32 ? steps_lo_i32 : steps_lo_f64));
    for (int64_t t0 = lo; t0 < hi; t0 += 32) {
      const int64_t l = t0 + lane;
      StageShift sh = {0, 0, 0, 0};
      if (l < hi) {
        const int64_t i = in.client_units[l], s = in.server_units[l];
        const int64_t u = in.up_units[l], d = in.down_units[l];
        sh.i = (int32_t)min(i, cap);
        sh.id = (int32_t)min(i + d, cap);
        sh.s = (int32_t)min(s, cap);
        sh.su = (int32_t)min(s + u, cap);
        shifts[l] = sh;
        const double r = in.r[l];
        // (g divides r and the quotient is below 2^31: the fp64 division is exact)
        rv[l] = mode == VM_INT32 ? (int64_t)__ddiv_rn(r, (double)g) : __double_as_longlong(r);
      }
      if (!reach) continue;
      if (trivial) {
        if (l < hi) reach[l] = make_int2(0, 0);
        continue;
      }
      const int cnt = (int)min((int64_t)32, hi - t0);
      int2 mine = make_int2(0, 0);
      for (int x = 0; x < cnt; ++x) {
        const int32_t si = __shfl_sync(0xffffffffu, sh.i, x), sid = __shfl_sync(0xffffffffu, sh.id, x);
        const int32_t ss = __shfl_sync(0xffffffffu, sh.s, x), ssu = __shfl_sync(0xffffffffu, sh.su, x);
        if (lane == x) mine = make_int2((int)min(mc, cap), (int)min(ms, cap));
        const int64_t nc = min(mc + si, ms + sid), ns = min(ms + ss, mc + ssu);
        mc = min(nc, cap);
        ms = min(ns, cap);
      }
      if (l < hi) reach[l] = mine;
    }
  }
}

// ---------------------------------------------------------------------------
// K2: DP stage kernels
//
// One instance = two budget-indexed rows C and S (W_eff + 1 columns) updated
// once per layer k (planner.py:128-143):
//   C_k[j] = r_k + max(C_{k-1}[j - i_k], S_{k-1}[j - i_k - d_k])
//   S_k[j] =       max(S_{k-1}[j - s_k], C_{k-1}[j - s_k - u_k])
// The dense variants hold the rows in different places:
//   * dp_stage_kernel<ROWS_SMEM=true>   one CTA, rows in its SMEM
//   * dp_stage_kernel<ROWS_SMEM=false>  one CTA, rows in global memory
//   * dp_stream_kernel (dp_stream.cuh)  a cluster, rows in L2-resident global memory
//   * dp_grid_kernel (dp_grid.cuh)      the whole GPU / capacity partitions
// (dp_steps.cuh holds the rows as breakpoint lists instead.)
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
  int32_t* overflow;  // [n] breakpoint-list kernel: 1 = a row exceeded its capacity
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

