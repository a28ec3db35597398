// K2 / K3 on breakpoint lists: the DP rows as monotone step functions.
//
// Fragment of sp_planner.cu: included there inside namespace sp::(anonymous),
// after the declarations it uses; not a standalone header.
//
// Every DP row is non-decreasing in the budget column j (a larger budget
// never hurts), and for model-derived instances it is a step function with
// few steps: the gpt2-24 rows of the benchmark (W_eff = 1e5 columns) take
// 7-130 distinct values (profiles/r02/steps/), because the achievable client
// values are sums over a handful of distinct layer costs.  A row is stored as
// its breakpoints -- (column, value) pairs with strictly increasing columns
// and values: row[j] = val[t] for col[t] <= j < col[t+1], unreachable (NEG)
// left of col[0] -- and one stage of planner.py:139-142
//   C_k[j] = r_k + max(C_{k-1}[j - i_k], S_{k-1}[j - i_k - d_k])
//   S_k[j] =       max(S_{k-1}[j - s_k], C_{k-1}[j - s_k - u_k])
// becomes two merges of shifted breakpoint lists: shifting a row moves its
// columns right (dropping those past W_eff), and the pointwise max of two
// non-decreasing step functions can only break where one of them does.
// Every value is produced by the same operations as the dense table (the max
// of the same two cells, then the same IEEE add of r_k), so the lists encode
// the dense tables exactly -- in every value domain except the
// NaN-propagating one, which stays on the dense kernels.
//
// Back-pointers.  _backtrace (planner.py:146-179) stays on a side at (k, j)
// iff the "stay" predecessor reproduces the stored value -- C: fl(C[k-1][j-i]
// + r) == C[k][j]; S: S[k-1][j-s] == S[k][j] -- and otherwise switches
// (outside the NaN domain the other predecessor then reproduces it).  Inside
// one breakpoint segment the stored value is constant and the stay
// predecessor is non-decreasing, so the predicate is false on a prefix of the
// segment and true on the rest: each breakpoint records `stay_from`, the
// first column of its segment where it holds (kNoStay: nowhere), found during
// the merge from the predecessor breakpoints the merge walks anyway.  The
// backtrack then needs ONE lookup per stage -- the breakpoint of the current
// row that covers j -- instead of re-deriving table values.
//
// Work decomposition: a group of G lanes per instance (G = 8: four instances
// per warp; G = 32 for the wide tier).  A merge splits the merged order of
// the two shifted lists into G equal diagonals (merge path: one binary search
// per lane); each lane walks its part sequentially keeping the events whose
// value differs from the previous one; a first pass counts them, a group scan
// places them, a second pass writes them.
//
// Store of one instance (read by the backtrack): (L+1) rows x {C, S}, each a
// count and CAP int2 {column, stay_from}, at a position the kernel computes
// itself -- (layer_off[k] + k) * steps_row_pair_bytes(CAP) -- in the
// device-planned tier (no host planning), or at DpWork::bp_off in the wave
// path:   cnt int32[(L+1) * 2] (16-B aligned) | ent int2[(L+1) * 2][CAP]
#pragma once

constexpr int kStepsCap = 192;       // tier 1: every instance, device-planned, a warp each
constexpr int kStepsCapWide = 1024;  // tier 2: instances tier 1 could not hold
constexpr int32_t kNoStay = INT32_MAX;

__host__ __device__ inline size_t steps_row_pair_bytes(int cap) { return 2 * (4 + (size_t)cap * 8); }
__host__ __device__ inline size_t steps_cnt_bytes(int L) { return (size_t)(L + 1) * 8; }  // keeps int2 8-B aligned
__host__ __device__ inline size_t steps_store_bytes(int L, int cap) {
  return steps_cnt_bytes(L) + (size_t)(L + 1) * 2 * cap * 8;
}

template <int MODE, typename V>
__device__ __forceinline__ V steps_max(V a, V b) {
  return a >= b ? a : b;  // np.maximum without NaN (the NaN domain never comes here)
}
template <int MODE, typename V>
__device__ __forceinline__ V steps_add(V a, V r) {
  if (MODE == VM_INT32) return a + r;  // exact: the domain's sums stay < 2^31
  else return dadd(a, r);
}

struct StepsArgs {
  const int64_t* layer_off;
  const uint8_t* sac;
  InstInfo* info;
  const StageShift* shifts;
  const int64_t* rv;
  const DpWork* work;          // wave path: instance and store offset (bp_off) per item; null: item = instance
  uint8_t* store;              // workspace base of the stores
  int32_t* flag;               // [n] device path: cleared once the instance is solved here (prep sets it)
  unsigned long long* solved;  // device path: [instances, DP cells, breakpoints stored, stages] solved here
  int32_t* overflow;           // wave path: [n] 1 = a row exceeded CAP
  int64_t n_items;
  int64_t max_cols;            // device path: wider instances are left to the dense kernels
  int64_t min_cols[2];         // device path, [int32, fp64 domain]: narrower ones too (one CTA's SMEM holds them)
};

template <int CAP>
__device__ __forceinline__ uint8_t* steps_store_of(const StepsArgs& a, int64_t item, int64_t inst) {
  return a.work ? a.store + a.work[item].bp_off
                : a.store + (size_t)(a.layer_off[inst] + inst) * steps_row_pair_bytes(CAP);
}

// first index in c[0, n) with c[idx] > x
__device__ __forceinline__ int upper_bound_i32(const int32_t* c, int n, int32_t x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int m = (lo + hi) >> 1;
    if (c[m] <= x) lo = m + 1;
    else hi = m;
  }
  return lo;
}

// One merge by a group of G lanes (g: lane in the group, gmask: the group's
// lanes): out = max(A shifted by ha, B shifted by hb) over columns <= W (+ r
// when ADD: the C row), with the stay_from of every kept breakpoint (A is the
// stay predecessor).  Writes the kept breakpoints to (oc, ov) in shared memory
// and their (column, stay_from) to `gent` in the store.  Returns the count, or
// -1 when it exceeds CAP.
//   1. merge path: lane g takes diagonal [ne*g/G, ne*(g+1)/G) of the merged
//      order (one binary search; an equal-column pair is never split);
//   2. it merges its part serially into the scratch (ec, ey) at the merged
//      positions -- every event carries the row value after it and whether
//      the stay predecessor reproduces that value (bit 31 of the column);
//      slots freed by merged equal-column pairs repeat the previous value;
//   3. a ballot compaction keeps the events whose value differs from the
//      previous slot's, and each kept event finds its segment's first stay
//      column by scanning the (short) run of events up to the next kept one.
template <int MODE, int G, int CAP, bool ADD, typename V>
__device__ __forceinline__ int steps_merge(const int32_t* ac, const V* av, int na, int ha, const int32_t* bc,
                                           const V* bv, int nb, int hb, int W, V rk, int32_t* ec, V* ey,
                                           int32_t* oc, V* ov, int2* gent, int g, uint32_t gmask) {
  const V NEG = VT<MODE>::neg();
  constexpr int32_t STAY = (int32_t)0x80000000u;
  constexpr int32_t COLM = 0x7fffffff;
  // columns <= W only: ballot counts over the sorted lists
  {
    int ca = 0, cb = 0;
    const int nmax = max(na, nb);
    for (int base = 0; base < nmax; base += G) {  // uniform trip count: every lane ballots
      const int x = base + g;
      ca += __popc(__ballot_sync(gmask, x < na && ac[x] <= W - ha));
      cb += __popc(__ballot_sync(gmask, x < nb && bc[x] <= W - hb));
    }
    na = ha > W ? 0 : ca;
    nb = hb > W ? 0 : cb;
  }
  const int ne = na + nb;
  int i0, j0;
  {
    const int d = (ne * g) / G;
    int lo = max(0, d - nb), hi = min(d, na);
    while (lo < hi) {
      const int m = (lo + hi) >> 1;
      if (ac[m] + ha <= bc[d - m - 1] + hb) lo = m + 1;
      else hi = m;
    }
    i0 = lo;
    j0 = d - lo;
    if (i0 > 0 && j0 < nb && ac[i0 - 1] + ha == bc[j0] + hb) ++j0;
  }
  int i1 = __shfl_down_sync(gmask, i0, 1, G), j1 = __shfl_down_sync(gmask, j0, 1, G);
  if (g == G - 1) {
    i1 = na;
    j1 = nb;
  }
  const int kend = g == G - 1 ? ne : (ne * (g + 1)) / G;
  V va = i0 > 0 ? av[i0 - 1] : NEG, vb = j0 > 0 ? bv[j0 - 1] : NEG;
  V y;
  {
    const V x = steps_max<MODE>(va, vb);
    y = (ADD && x != NEG) ? steps_add<MODE>(x, rk) : x;
  }
  int i = i0, j = j0, k = (ne * g) / G;
  int cA = i < i1 ? ac[i] + ha : COLM, cB = j < j1 ? bc[j] + hb : COLM;
  V nA = i < i1 ? av[i] : NEG, nB = j < j1 ? bv[j] : NEG;
  while (i < i1 || j < j1) {
    const bool tA = cA <= cB, tB = cB <= cA;
    const int col = tA ? cA : cB;
    if (tA) {
      va = nA;
      ++i;
      cA = i < i1 ? ac[i] + ha : COLM;
      nA = i < i1 ? av[i] : nA;
    }
    if (tB) {
      vb = nB;
      ++j;
      cB = j < j1 ? bc[j] + hb : COLM;
      nB = j < j1 ? bv[j] : nB;
    }
    const V x = steps_max<MODE>(va, vb);
    y = ADD ? steps_add<MODE>(x, rk) : x;
    const bool stay = va != NEG && (ADD ? steps_add<MODE>(va, rk) == y : va == y);
    ec[k] = stay ? (col | STAY) : col;
    ey[k] = y;
    ++k;
  }
  for (; k < kend; ++k) {  // freed by merged pairs: the value continues, no event
    ec[k] = COLM;
    ey[k] = y;
  }
  __syncwarp(gmask);
  const uint32_t below = (1u << (threadIdx.x & 31)) - 1u;
  int total = 0;
  for (int base = 0; base < ne; base += G) {
    const int e = base + g;
    bool keep = false;
    int32_t c = COLM;
    V v = NEG;
    if (e < ne) {
      c = ec[e];
      v = ey[e];
      keep = e == 0 ? v != NEG : v != ey[e - 1];
    }
    const uint32_t m = __ballot_sync(gmask, keep);
    const int pos = total + __popc(m & below);
    if (keep && pos < CAP) {
      const int col = c & COLM;
      oc[pos] = col;
      ov[pos] = v;
      // first stay column of this breakpoint's segment: this event or a later
      // one before the next kept event
      int32_t sf = kNoStay;
      for (int f = e; f < ne; ++f) {
        const int32_t cf = ec[f];
        if (f > e && ey[f] != ey[f - 1]) break;
        if (cf & STAY) {
          sf = cf & COLM;
          break;
        }
      }
      gent[pos] = make_int2(col, sf);
    }
    total += __popc(m);
  }
  __syncwarp(gmask);
  return total > CAP ? -1 : total;
}

// lists of CAP entries per instance in shared memory: rows [2 bufs][C|S] +
// the merge scratch [2 CAP].  (A two-pass merge without the scratch -- 4
// lists, more resident warps -- measured slower: 2.43 vs 1.84 ms at CAP 256.)
constexpr int kStepsArrays = 6;

// One group of G lanes per instance, WPB warps per block; rows double-buffered
// in the group's shared memory, every row's (column, stay_from) written to the
// instance's store.  Device path (a.work == null): group k takes instance k if
// it is in this kernel's value domain and min_cols <= W_eff + 1 < max_cols.
template <int MODE, int CAP, int G, int WPB>
__global__ void __launch_bounds__(WPB * 32) dp_steps_kernel(StepsArgs a) {
  using V = typename VT<MODE>::T;
  constexpr int GPW = 32 / G;                                        // groups (instances) per warp
  constexpr size_t INST_BYTES = (size_t)kStepsArrays * CAP * (4 + sizeof(V));  // rows [2 bufs][C|S] (+ merge scratch)
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / G, g = lane % G;
  const uint32_t gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (grp * G));
  const int64_t item = ((int64_t)blockIdx.x * WPB + warp) * GPW + grp;
  if (item >= a.n_items) return;  // whole groups leave together
  const int64_t inst = a.work ? a.work[item].inst : item;
  const InstInfo inf = a.info[inst];
  if (!a.work && (inf.mode != MODE || inf.w_eff + 1 >= a.max_cols ||
                  inf.w_eff + 1 < a.min_cols[MODE == VM_INT32 ? 0 : 1]))
    return;
  unsigned char* ws = smem + (size_t)(warp * GPW + grp) * INST_BYTES;
  int32_t* rc = reinterpret_cast<int32_t*>(ws);    // [2][2][CAP]
  V* rvv = reinterpret_cast<V*>(ws + 4 * CAP * 4);  // [2][2][CAP]
  int32_t* ecs = reinterpret_cast<int32_t*>(ws + 4 * CAP * (4 + sizeof(V)));            // [2 CAP]
  V* eys = reinterpret_cast<V*>(ws + 4 * CAP * (4 + sizeof(V)) + 2 * CAP * 4);         // [2 CAP]
  auto rcol = [&](int buf, int row) { return rc + (buf * 2 + row) * CAP; };
  auto rval = [&](int buf, int row) { return rvv + (buf * 2 + row) * CAP; };

  const int64_t lo = a.layer_off[inst];
  const int L = (int)(a.layer_off[inst + 1] - lo);
  const int W = (int)inf.w_eff;
  const bool sac = a.sac[inst] != 0;
  uint8_t* st = steps_store_of<CAP>(a, item, inst);
  int32_t* g_cnt = reinterpret_cast<int32_t*>(st);
  int2* g_ent = reinterpret_cast<int2*>(st + steps_cnt_bytes(L));

  // row 0: the origin side holds +0 everywhere, the other side nothing
  int nC = sac ? 1 : 0, nS = sac ? 0 : 1;
  if (g == 0) {
    rcol(0, 0)[0] = 0;
    rval(0, 0)[0] = V(0);
    rcol(0, 1)[0] = 0;
    rval(0, 1)[0] = V(0);
    g_cnt[0] = nC;
    g_cnt[1] = nS;
    g_ent[0] = make_int2(0, kNoStay);
    g_ent[CAP] = make_int2(0, kNoStay);
  }
  __syncwarp(gmask);
  int buf = 0;
  bool over = false;
  unsigned long long stored = (unsigned long long)(nC + nS);
  // stage records one stage ahead: their load latency overlaps the merges
  StageShift sh_next = a.shifts[lo];
  int64_t bits_next = a.rv[lo];
  for (int t = 0; t < L; ++t) {
    const StageShift sh = sh_next;
    const int64_t bits = bits_next;
    if (t + 1 < L) {
      sh_next = a.shifts[lo + t + 1];
      bits_next = a.rv[lo + t + 1];
    }
    const V rk = MODE == VM_INT32 ? (V)(int32_t)bits : (V)__longlong_as_double(bits);
    const int nb = buf ^ 1;
    const size_t r0 = (size_t)(t + 1) * 2;
    const int nC2 = steps_merge<MODE, G, CAP, true, V>(rcol(buf, 0), rval(buf, 0), nC, sh.i, rcol(buf, 1),
                                                       rval(buf, 1), nS, sh.id, W, rk, ecs, eys, rcol(nb, 0),
                                                       rval(nb, 0), g_ent + r0 * CAP, g, gmask);
    const int nS2 = steps_merge<MODE, G, CAP, false, V>(rcol(buf, 1), rval(buf, 1), nS, sh.s, rcol(buf, 0),
                                                        rval(buf, 0), nC, sh.su, W, rk, ecs, eys, rcol(nb, 1),
                                                        rval(nb, 1), g_ent + (r0 + 1) * CAP, g, gmask);
    if (nC2 < 0 || nS2 < 0) {
      over = true;
      break;
    }
    nC = nC2;
    nS = nS2;
    stored += (unsigned long long)(nC + nS);
    buf = nb;
    if (g == 0) {
      g_cnt[r0] = nC;
      g_cnt[r0 + 1] = nS;
    }
    __syncwarp(gmask);
  }
  if (g == 0) {
    if (a.overflow) a.overflow[inst] = over ? 1 : 0;
    if (!over) {
      // value at column W: the last breakpoint (every stored column is <= W)
      const V NEG = VT<MODE>::neg();
      const V ec_ = nC > 0 ? rval(buf, 0)[nC - 1] : NEG;
      const V es_ = nS > 0 ? rval(buf, 1)[nS - 1] : NEG;
      a.info[inst].end_c = to_f64(ec_, inf.scale);
      a.info[inst].end_s = to_f64(es_, inf.scale);
      if (a.flag) a.flag[inst] = 0;
      if (a.solved) {
        atomicAdd(a.solved, 1ull);
        atomicAdd(a.solved + 1, (unsigned long long)L * (unsigned long long)(W + 1));  // DP cells solved
        atomicAdd(a.solved + 2, stored);
        atomicAdd(a.solved + 3, (unsigned long long)L);
      }
    }
  }
}

// K3 on breakpoint lists: end-side argmax (planner.py:190-200) and the walk
// of planner.py:146-179 -- per stage, the breakpoint of the current row that
// covers j decides stay (j >= stay_from) or switch -- then _finish.  One group
// of G lanes per instance; a lookup is a G-ary search (G independent loads
// per round).  Device path: instances whose flag is still set are left
// alone; wave path: overflowed ones.  Value-free: one launch serves every
// value domain.
constexpr int kBtSmemStages = 255;  // row counts of instances up to this many stages sit in shared memory

template <int CAP, int G, int WPB>
__global__ void __launch_bounds__(WPB * 32) backtrack_steps_kernel(sp_instances in, StepsArgs a,
                                                                   int32_t* idx_scratch, sp_policies out) {
  constexpr int GPW = 32 / G;
  __shared__ int32_t scnt[WPB * GPW][2 * (kBtSmemStages + 1)];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / G, g = lane % G;
  const uint32_t gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (grp * G));
  const int64_t item = ((int64_t)blockIdx.x * WPB + warp) * GPW + grp;
  if (item >= a.n_items) return;
  const int64_t inst = a.work ? a.work[item].inst : item;
  if (a.work ? a.overflow[inst] != 0 : a.flag[inst] != 0) return;
  const InstInfo inf = a.info[inst];
  const int64_t lo = in.layer_off[inst];
  const int L = (int)(in.layer_off[inst + 1] - lo);
  double ec = inf.end_c, es = inf.end_s;
  const int8_t must = in.must_end_at ? in.must_end_at[inst] : (int8_t)-1;
  if (must == 1) es = -INFINITY;
  else if (must == 0) ec = -INFINITY;
  const double pmax = (es > ec) ? es : ec;  // Python builtin max(end_c, end_s)
  uint8_t* pi = out.pi + lo;
  if (pmax == -INFINITY) {  // _infeasible
    if (g == 0) {
      for (int k = 0; k < L; ++k) pi[k] = 0;
      finish_policy(in, inst, lo, L, idx_scratch + lo, out, true, false);
      out.status[inst] = SP_OK;
    }
    return;
  }
  const uint8_t* st = steps_store_of<CAP>(a, item, inst);
  const int32_t* g_cnt = reinterpret_cast<const int32_t*>(st);
  const int2* g_ent = reinterpret_cast<const int2*>(st + steps_cnt_bytes(L));
  if (L <= kBtSmemStages) {  // the row counts once, instead of one dependent load per step
    int32_t* sc = scnt[warp * GPW + grp];
    for (int x = g; x < 2 * (L + 1); x += G) sc[x] = g_cnt[x];
    __syncwarp(gmask);
    g_cnt = sc;
  }
  bool client = ec >= es;
  int64_t j = inf.w_eff;
  int32_t status = SP_OK;
  StageShift sh_next = a.shifts[lo + L - 1];
  for (int k = L; k >= 1; --k) {
    const StageShift sh = sh_next;
    if (k > 1) sh_next = a.shifts[lo + k - 2];
    const size_t r = (size_t)k * 2 + (client ? 0 : 1);
    const int2* ent = g_ent + r * CAP;
    // G-ary search for the number of breakpoints at or left of j
    int lo_i = 0, hi_i = g_cnt[r];  // the count lies in [lo_i, hi_i]
    while (lo_i < hi_i) {
      const int span = hi_i - lo_i;
      const int step = (span + G) / (G + 1);
      const int p = lo_i + (g + 1) * step - 1;  // this lane's pivot
      const bool valid = p < hi_i;
      const int c = __popc(__ballot_sync(gmask, valid && ent[p].x <= j));  // pivots <= j: a prefix
      const int nv = __popc(__ballot_sync(gmask, valid));
      const int nlo = lo_i + c * step;
      hi_i = c < nv ? lo_i + (c + 1) * step - 1 : hi_i;
      lo_i = nlo;
    }
    if (lo_i == 0) {  // j left of the row's first breakpoint: unreachable
      status = SP_ERR_BACKTRACE;
      break;
    }
    const bool stay = j >= ent[lo_i - 1].y;
    if (client) {
      if (g == 0) pi[k - 1] = 1;
      j -= stay ? sh.i : sh.id;
      client = stay;
    } else {
      if (g == 0) pi[k - 1] = 0;
      j -= stay ? sh.s : sh.su;
      client = !stay;
    }
    if (j < 0) {  // no predecessor reproduces the value (planner.py:168-169 / 177-178)
      status = SP_ERR_BACKTRACE;
      break;
    }
  }
  __syncwarp(gmask);
  if (g != 0) return;
  out.status[inst] = status;
  if (status != SP_OK) return;
  finish_policy(in, inst, lo, L, idx_scratch + lo, out, false, false);
}
