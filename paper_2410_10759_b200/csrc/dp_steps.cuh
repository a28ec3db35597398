// K2 + K3 on breakpoint lists: the DP rows as monotone step functions.
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
// the merge from the predecessor events the merge produces anyway.  The
// backtrack then needs ONE lookup per stage -- the breakpoint of the current
// row that covers j -- instead of re-deriving table values.
//
// Work decomposition: one warp per instance; the two merges of a stage run
// side by side, half-warp 0 building the C row and half-warp 1 the S row,
// in lockstep (every ballot and shuffle is full-warp), so a stage costs one
// merge's latency chain.  A merge splits
// the merged order of its two shifted lists into 16 equal diagonals (merge
// path, one binary search per lane); each lane merges its part serially into
// a scratch array at the merged positions -- every event carries the row
// value after it and whether the stay predecessor reproduces it -- counting
// the events it keeps (value differs from the previous slot's); a scan of
// the counts places them, and each lane writes its kept breakpoints with
// their stay_from.  The new row overwrites the old one (both merges have
// finished reading the old rows by then), so shared memory holds
// two rows and two scratch arrays per instance.
//
// The same warp then walks the instance back (end-side choice, planner.py:
// 182-202; _backtrace, planner.py:146-179) through the rows it has just
// stored -- the stage records and the breakpoints of both candidate rows are
// fetched kWalkDepth stages ahead, as whole 16-B breakpoint pairs (a row of
// odd count carries a written padding entry) -- and computes _finish
// (planner.py:88-101) with the placement and the compacted r values in shared
// memory.
//
// Store of one instance (read by the walk): (L+1) rows x {C, S}, each a count
// and CAP int2 {column, stay_from}, at a position the kernel computes itself
// -- (layer_off[k] + k - pos0) * steps_row_pair_bytes(CAP) -- in the
// device-planned tier (no host planning; a batch whose stores do not fit the
// workspace runs in waves of consecutive instances), or at DpWork::bp_off in
// the host-planned path:
//   cnt int32[(L+1) * 2] (padded to 16 B) | ent int2[(L+1) * 2][CAP]
#pragma once

constexpr int kStepsCap = 192;       // tier 1: every instance, device-planned, a warp each
constexpr int kStepsCapWide = 1024;  // tier 2: instances tier 1 could not hold
constexpr int32_t kNoStay = INT32_MAX;

// sizes keep every store, and every row in it, 16-B aligned (the walk copies
// breakpoint pairs with 16-B cp.async; CAP is even)
__host__ __device__ inline size_t steps_row_pair_bytes(int cap) { return 16 + (size_t)cap * 16; }
__host__ __device__ inline size_t steps_cnt_bytes(int L) { return ((size_t)(L + 1) * 8 + 15) & ~(size_t)15; }
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
  int32_t* idx;                // [total_layers] scratch of _finish for instances too long for shared memory
  int64_t n_items;
  int64_t item0, pos0;         // device path: instances [item0, item0 + n_items); store of instance k at
                               // (layer_off[k] + k - pos0) row pairs (pos0 = layer_off[item0] + item0)
  int64_t max_cols;            // device path: wider instances are left to the dense kernels
  int64_t min_cols[2];         // device path, [int32, fp64 domain]: narrower ones too (one CTA's SMEM holds them)
  int32_t walk;                // 1: walk back and finish every solved instance (the policies below)
  sp_instances in;
  sp_policies out;
};

template <int CAP>
__device__ __forceinline__ uint8_t* steps_store_of(const StepsArgs& a, int64_t item, int64_t inst) {
  return a.work ? a.store + a.work[item].bp_off
                : a.store + (size_t)(a.layer_off[inst] + inst - a.pos0) * steps_row_pair_bytes(CAP);
}

constexpr uint32_t kFull = 0xffffffffu;

// A breakpoint (or a merge event) in shared memory: column and row value
// side by side, one 8-B (int32 domain) or 16-B (fp64) access.
template <int MODE> struct Ent;
template <> struct __align__(8) Ent<VM_INT32> {
  int32_t c;
  int32_t v;
};
template <> struct __align__(16) Ent<VM_F64> {
  int32_t c;
  int32_t pad;
  double v;
};
template <int MODE, typename V>
__device__ __forceinline__ Ent<MODE> mk_ent(int32_t c, V v) {
  Ent<MODE> e;
  e.c = c;
  e.v = v;
  return e;
}

// One merge by the 16 lanes of half-warp h (g: lane in the half), run by both
// halves at once: out = max(A shifted by ha, B shifted by hb) over columns
// <= W, plus rk (0 for the S row: the add is exact then) on reachable values,
// with the stay_from of every kept breakpoint (A is the stay predecessor).
// na / nb: the breakpoints of A / B at columns <= W - ha / W - hb (counted
// by the previous stage's write pass).  Writes the kept breakpoints to `out`
// in shared memory -- this half's old row: the old rows are dead once the
// merge phase is over -- and their (column, stay_from) to `gent` in the
// store.  Returns the count (or -1 when it exceeds CAP) and, for the next
// stage, the new row's breakpoints at columns <= t1 / <= t2 (cnt1 / cnt2).
//   1. merge path: lane g takes diagonal [ne*g/16, ne*(g+1)/16) of the merged
//      order (one binary search; an equal-column pair is never split), and
//      merges its part serially into its region of the scratch (from its
//      diagonal's start) -- every event carries the row value after it and
//      whether the stay predecessor reproduces that value (bit 31 of the
//      column); a merged equal-column pair is one event.  An event is
//      kept iff its value differs from the previous slot's; the lane knows
//      the value before its part, so it counts its own;
//   2. a scan of the counts over the half places every lane's kept events;
//   3. each lane re-reads its part and writes its kept breakpoints (a
//      warp-uniform trip count with predicated updates: the data-dependent
//      loop's reconvergence cost 8 % of the kernel); a kept breakpoint's
//      stay_from is the column of the first stay event from it up to the
//      next kept one -- in the lane's own part, or in the first later part
//      holding a kept or a stay event (one ballot).
template <int MODE, int CAP, typename V>
__device__ __forceinline__ int steps_merge_half(const Ent<MODE>* A, int na, int ha, const Ent<MODE>* B, int nb,
                                                int hb, V rk, Ent<MODE>* ev, Ent<MODE>* out, int2* gent, int g,
                                                int h, int t1, int t2, int& cnt1, int& cnt2) {
  const V NEG = VT<MODE>::neg();
  constexpr int32_t STAY = (int32_t)0x80000000u;
  constexpr int32_t COLM = 0x7fffffff;
  const int hs = h << 4;
  // 1. merge path + serial merge into the scratch
  const int ne = na + nb;
  const int k0 = (ne * g) >> 4;
  int i0, j0;
  {
    int lo = max(0, k0 - nb), hi = min(k0, na);
    while (lo < hi) {
      const int m = (lo + hi) >> 1;
      if (A[m].c + ha <= B[k0 - m - 1].c + hb) lo = m + 1;
      else hi = m;
    }
    i0 = lo;
    j0 = k0 - lo;
    if (i0 > 0 && j0 < nb && A[i0 - 1].c + ha == B[j0].c + hb) ++j0;
  }
  int i1 = __shfl_down_sync(kFull, i0, 1, 16), j1 = __shfl_down_sync(kFull, j0, 1, 16);
  if (g == 15) {
    i1 = na;
    j1 = nb;
  }
  V y0;             // the row value just before this lane's part
  int nk = 0;       // kept events in this lane's part
  int kev;          // end of this lane's events in the scratch (k0 + events)
  {
    V va = i0 > 0 ? A[i0 - 1].v : NEG, vb = j0 > 0 ? B[j0 - 1].v : NEG;
    {
      const V x = steps_max<MODE>(va, vb);
      y0 = x != NEG ? steps_add<MODE>(x, rk) : x;
    }
    V y = y0;
    int i = i0, j = j0, k = k0;
    // branch-free: both lists are re-read at clamped positions every event
    // (a position past the lane's range reads as column COLM)
    const int ilast = max(i1 - 1, 0), jlast = max(j1 - 1, 0);
    Ent<MODE> ea = A[min(i, ilast)], eb = B[min(j, jlast)];
    int cA = i < i1 ? ea.c + ha : COLM, cB = j < j1 ? eb.c + hb : COLM;
    while (min(cA, cB) != COLM) {
      const bool tA = cA <= cB, tB = cB <= cA;
      const int col = min(cA, cB);
      va = tA ? ea.v : va;
      vb = tB ? eb.v : vb;
      i += tA ? 1 : 0;
      j += tB ? 1 : 0;
      ea = A[min(i, ilast)];
      eb = B[min(j, jlast)];
      cA = i < i1 ? ea.c + ha : COLM;
      cB = j < j1 ? eb.c + hb : COLM;
      // after an event one side holds a breakpoint value: the max is reachable
      const V yn = steps_add<MODE>(steps_max<MODE>(va, vb), rk);
      // (int32: the add is exact, so va + rk == max(va, vb) + rk iff va >= vb)
      const bool stay = va != NEG && (MODE == VM_INT32 ? va >= vb : steps_add<MODE>(va, rk) == yn);
      const bool keep = yn != y;
      nk += keep ? 1 : 0;
      ev[k] = mk_ent<MODE>(stay ? (col | STAY) : col, yn);
      y = yn;
      ++k;
    }
    kev = k;  // (a merged equal-column pair is one event: fewer events than merged positions)
  }
  // 2. output positions (a scan of the kept counts over the half)
  int incl = nk;
#pragma unroll
  for (int o = 1; o < 16; o <<= 1) {
    const int t = __shfl_up_sync(kFull, incl, o, 16);
    if (g >= o) incl += t;
  }
  const int total = __shfl_sync(kFull, incl, hs + 15);
  __syncwarp(kFull);  // both halves are done reading the old rows
  // 3. this lane writes its kept breakpoints: the new row (over the old one)
  // and (column, stay_from) to the store; it counts the ones at columns
  // <= t1 / t2 for the next stage's clip
  int c1 = 0, c2 = 0;
  {
    int pos = incl - nk, open = -1;
    int32_t ocol = 0, osf = kNoStay;  // the open breakpoint: column, stay_from found so far
    int32_t fs_pre = kNoStay;  // first stay event of this part before its first kept one
    V prev = y0;
    // (warp-uniform trip count, every update predicated)
    const int nev = kev - k0;
    const int trips = (int)__reduce_max_sync(kFull, (uint32_t)nev);
    for (int it = 0; it < trips; ++it) {
      const bool act = it < nev;
      const Ent<MODE> e = ev[k0 + min(it, max(nev - 1, 0))];
      const int32_t col = e.c & COLM;
      const bool keep = act && e.v != prev;  // kept: the previous open breakpoint is complete
      if (keep && (unsigned)open < (unsigned)CAP) gent[open] = make_int2(ocol, osf);
      if (keep) out[pos] = mk_ent<MODE>(col, e.v);  // (pos < 2 CAP: past CAP only on overflow, inside this warp's region)
      fs_pre = (keep && open < 0) ? osf : fs_pre;
      open = keep ? pos : open;
      ocol = keep ? col : ocol;
      osf = keep ? kNoStay : osf;
      pos += keep ? 1 : 0;
      c1 += (keep && col <= t1) ? 1 : 0;
      c2 += (keep && col <= t2) ? 1 : 0;
      osf = (act && e.c < 0 && osf == kNoStay) ? col : osf;  // bit 31: a stay event
      prev = act ? e.v : prev;
    }
    if (open < 0) fs_pre = osf;
    // the stay_from of a segment running past this lane's part: the first
    // later lane with a kept event or an earlier stay event decides it
    const uint32_t T = (__ballot_sync(kFull, nk > 0 || fs_pre != kNoStay) >> hs) & 0xffffu;
    const uint32_t nxt = g == 15 ? 0u : (T >> (g + 1)) << (g + 1);
    const int32_t tail_in = __shfl_sync(kFull, fs_pre, hs + (nxt ? __ffs(nxt) - 1 : g));
    const int32_t tail_sf = nxt ? tail_in : kNoStay;
    if (open >= 0 && open < CAP) gent[open] = make_int2(ocol, osf != kNoStay ? osf : tail_sf);
  }
  // a row of odd count gets a padding entry, so the walk's 16-B pair copies
  // only ever read written memory
  if (g == 15 && (total & 1) && total < CAP) gent[total] = make_int2(COLM, kNoStay);
  // the half's sums, both halves in one reduction each (counts < 2^16)
  cnt1 = __reduce_add_sync(kFull, (uint32_t)c1 << hs);
  cnt2 = __reduce_add_sync(kFull, (uint32_t)c2 << hs);
  cnt1 = (int)(((uint32_t)cnt1 >> hs) & 0xffffu);
  cnt2 = (int)(((uint32_t)cnt2 >> hs) & 0xffffu);
  __syncwarp(kFull);
  return total > CAP ? -1 : total;
}

// numpy-order _finish (planner.py:88-101) of a placement held in shared
// memory by the whole warp: exact integer latency (any order), the placement
// to global memory, r compacted into client / server order in `buf`, then the
// two numpy pairwise sums (np_sum, one lane, shared-memory operands).
__device__ __forceinline__ void finish_policy_warp(const sp_instances& in, int64_t inst, int64_t lo, int L,
                                                   const uint8_t* pis, double* buf, const sp_policies& out,
                                                   bool infeasible, int lane) {
  const bool sac = in.source_at_client[inst] != 0;
  const uint32_t below = (1u << lane) - 1u;
  long long lat = 0;
  int n1 = 0;
  for (int base = 0; base < L; base += 32) {
    const int k = base + lane;
    const bool v = k < L;
    const int x = v ? pis[k] : 0;
    if (v) {
      const int prev = k == 0 ? (sac ? 1 : 0) : pis[k - 1];
      lat += x ? in.client_units[lo + k] + (prev == 0 ? in.down_units[lo + k] : 0)
               : in.server_units[lo + k] + (prev == 1 ? in.up_units[lo + k] : 0);
      out.pi[lo + k] = (uint8_t)x;
    }
    n1 += __popc(__ballot_sync(kFull, v && x));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lat += __shfl_xor_sync(kFull, lat, o);
  int a = 0, b = n1;
  for (int base = 0; base < L; base += 32) {
    const int k = base + lane;
    const bool v = k < L;
    const int x = v ? pis[k] : 0;
    const uint32_t bc = __ballot_sync(kFull, v && x), bs = __ballot_sync(kFull, v && !x);
    if (v) buf[x ? a + __popc(bc & below) : b + __popc(bs & below)] = in.r[lo + k];
    a += __popc(bc);
    b += __popc(bs);
  }
  __syncwarp(kFull);
  if (lane == 0) {
    out.client_value[inst] = np_sum([&](int64_t m) { return buf[m]; }, n1);
    out.server_load[inst] = np_sum([&](int64_t m) { return buf[n1 + m]; }, L - n1);
    out.integer_latency[inst] = (int64_t)lat;
    out.feasible[inst] = infeasible ? 0 : ((int64_t)lat <= in.budget[inst] ? 1 : 0);
    out.status[inst] = SP_OK;
  }
}

// entries per instance in shared memory: rows [C|S] + the two merges'
// events [2][EV x CAP] (EV = 2 holds any merge of two rows of CAP; EV = 1
// halves the footprint, a merge of more than CAP events overflows to the next
// tier; the wide tier keeps 2)
#ifndef SP_STEPS_EV2
#define SP_STEPS_EV2 4  // twice the events scratch per half, in units of CAP (4: 2 CAP)
#endif
#ifndef SP_STEPS_MINB
#define SP_STEPS_MINB 8
#endif
template <int CAP> __host__ __device__ constexpr int steps_ev2() { return CAP >= 1024 ? 4 : SP_STEPS_EV2; }
// entries per instance: 2 rows + 2 halves x EV2/2 x CAP events
template <int CAP> __host__ __device__ constexpr int steps_arrays() { return 2 + steps_ev2<CAP>(); }
__host__ __device__ inline int steps_arrays_rt(int cap) { return 2 + (cap >= 1024 ? 4 : SP_STEPS_EV2); }
template <int CAP, typename E> __host__ __device__ constexpr int walk_depth() {
  // as many prefetched stages (at most 8) as the instance's shared memory holds
  // next to the placement and the row counts of a 128-stage instance
  return (int)(((size_t)steps_arrays<CAP>() * CAP * sizeof(E) - 128 - 272) / (32 + 2 * 64 * 8)) >= 8
             ? 8
             : (int)(((size_t)steps_arrays<CAP>() * CAP * sizeof(E) - 128 - 272) / (32 + 2 * 64 * 8));
}
constexpr size_t kWalkSlot = 32 + 2 * 64 * 8;

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
// 16-B slot, `bytes` (0, 8 or 16) of them copied, the rest zero-filled: one
// instruction for every lane instead of a divergent choice of copy sizes
__device__ __forceinline__ void cp_async16_part(void* dst, const void* src, int bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// One warp per instance, WPB warps per block: forward pass over the
// breakpoint lists, every row's (column, stay_from) written to the
// instance's store, then (a.walk) the walk back and _finish.  Device path
// (a.work == null): warp k takes instance k if it is in this kernel's value
// domain and min_cols <= W_eff + 1 < max_cols; an instance whose rows outgrow
// CAP keeps its flag (device path) / gets its overflow bit (wave path) and
// is left to the next tier.
template <int MODE, int CAP, int WPB>
__global__ void __launch_bounds__(WPB * 32, WPB == 1 ? 1 : SP_STEPS_MINB) dp_steps_kernel(StepsArgs a) {
  using V = typename VT<MODE>::T;
  using E = Ent<MODE>;
  constexpr size_t INST_BYTES = (size_t)steps_arrays<CAP>() * CAP * sizeof(E);
  constexpr int EVC = steps_ev2<CAP>() * CAP / 2;  // merge events per half
  constexpr int kWalkDepth = walk_depth<CAP, E>();
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = lane >> 4, g = lane & 15;
  const int64_t item = (int64_t)blockIdx.x * WPB + warp;
  if (item >= a.n_items) return;  // whole warps leave together
  const int64_t inst = a.work ? a.work[item].inst : a.item0 + item;
  const InstInfo inf = a.info[inst];
  if (!a.work && (inf.mode != MODE || inf.w_eff + 1 >= a.max_cols ||
                  inf.w_eff + 1 < a.min_cols[MODE == VM_INT32 ? 0 : 1]))
    return;
  unsigned char* ws = smem + (size_t)warp * INST_BYTES;
  E* rows = reinterpret_cast<E*>(ws);              // [2 rows: C, S][CAP]
  E* evs = rows + 2 * CAP;                         // [2 halves][EVC] merge events

  const int64_t lo = a.layer_off[inst];
  const int L = (int)(a.layer_off[inst + 1] - lo);
  const int W = (int)inf.w_eff;
  const bool sac = a.sac[inst] != 0;
  uint8_t* st = steps_store_of<CAP>(a, item, inst);
  int32_t* g_cnt = reinterpret_cast<int32_t*>(st);
  int2* g_ent = reinterpret_cast<int2*>(st + steps_cnt_bytes(L));

  // row 0: the origin side holds +0 everywhere, the other side nothing
  const int n0 = (h == 0) == sac ? 1 : 0;  // breakpoints of row h (C for h = 0)
  if (g == 0) {
    rows[h * CAP] = mk_ent<MODE>(0, V(0));
    g_cnt[h] = n0;
    g_ent[h * CAP] = make_int2(0, kNoStay);
    g_ent[h * CAP + 1] = make_int2(0x7fffffff, kNoStay);  // the pair's padding entry
  }
  __syncwarp(kFull);
  bool over = false;
  unsigned long long stored = 1;
  int nMine = n0;  // breakpoints of row h
  // stage records one stage ahead: their load latency overlaps the merges
  StageShift sh = a.shifts[lo];
  int64_t bits = a.rv[lo];
  // clipped counts of this stage's two lists (row 0: the one breakpoint at column 0)
  int na = (n0 && (h ? sh.s : sh.i) <= W) ? 1 : 0;
  int nb = (!n0 && (h ? sh.su : sh.id) <= W) ? 1 : 0;
  for (int t = 0; t < L; ++t) {
    StageShift sh_next = sh;
    int64_t bits_next = bits;
    if (t + 1 < L) {
      sh_next = a.shifts[lo + t + 1];
      bits_next = a.rv[lo + t + 1];
    }
    const V rk = h ? V(0) : (MODE == VM_INT32 ? (V)(int32_t)bits : (V)__longlong_as_double(bits));
    const size_t r0 = (size_t)(t + 1) * 2;
    // next stage's clip thresholds of the row this half builds: as its own
    // merge's A (C: i, S: s) and as the other merge's B (C: s + u, S: i + d)
    const int t1 = W - (h ? sh_next.s : sh_next.i), t2 = W - (h ? sh_next.id : sh_next.su);
    if (EVC < 2 * CAP && __any_sync(kFull, na + nb > EVC)) {  // more events than the scratch holds
      over = true;
      break;
    }
    int c1, c2;
    const int n2 = steps_merge_half<MODE, CAP, V>(rows + h * CAP, na, h ? sh.s : sh.i, rows + (1 - h) * CAP, nb,
                                                  h ? sh.su : sh.id, rk, evs + h * EVC, rows + h * CAP,
                                                  g_ent + (r0 + h) * CAP, g, h, t1, t2, c1, c2);
    const int n2o = __shfl_xor_sync(kFull, n2, 16);
    if (n2 < 0 || n2o < 0) {
      over = true;
      break;
    }
    nMine = n2;
    na = c1;
    nb = __shfl_xor_sync(kFull, c2, 16);
    stored += (unsigned long long)n2;  // this half's row (summed over both halves below)
    if (g == 0) g_cnt[r0 + h] = n2;
    sh = sh_next;
    bits = bits_next;
    __syncwarp(kFull);
  }
  stored += __shfl_xor_sync(kFull, stored, 16) - 1;  // both rows of every stage (+ the origin row)
  const int nC = h == 0 ? nMine : __shfl_xor_sync(kFull, nMine, 16);
  const int nS = h == 1 ? nMine : __shfl_xor_sync(kFull, nMine, 16);
  if (a.overflow && lane == 0) a.overflow[inst] = over ? 1 : 0;
  if (over) return;
  // value at column W: the last breakpoint (every stored column is <= W)
  const V NEG = VT<MODE>::neg();
  const double end_c = to_f64(nC > 0 ? rows[nC - 1].v : NEG, inf.scale);
  const double end_s = to_f64(nS > 0 ? rows[CAP + nS - 1].v : NEG, inf.scale);
  if (lane == 0) {
    a.info[inst].end_c = end_c;
    a.info[inst].end_s = end_s;
    if (a.flag) a.flag[inst] = 0;
    if (a.solved) {
      atomicAdd(a.solved, 1ull);
      atomicAdd(a.solved + 1, (unsigned long long)L * (unsigned long long)(W + 1));  // DP cells solved
      atomicAdd(a.solved + 2, stored);
      atomicAdd(a.solved + 3, (unsigned long long)L);
    }
  }
  if (!a.walk) return;

  // ---- the walk back: end side (planner.py:182-202), _backtrace (146-179)
  double ec = end_c, es = end_s;
  const int8_t must = a.in.must_end_at ? a.in.must_end_at[inst] : (int8_t)-1;
  if (must == 1) es = -INFINITY;
  else if (must == 0) ec = -INFINITY;
  const double pmax = (es > ec) ? es : ec;  // Python builtin max(end_c, end_s)
  // The walk runs out of the warp's shared memory, free now: the placement
  // (L bytes), then a ring of kWalkDepth stages fetched ahead with cp.async
  // -- the stage record, the row counts and the first 64 breakpoints of both
  // rows of a stage -- so the L2 latency of the store stays off the chain of
  // dependent lookups; _finish then reuses the ring for the r values.
  // Instances too long for that walk with plain loads, placement in global.
  // The row counts of every stage are copied into shared memory first (the
  // forward pass left them in the store, L2-hot), so each stage's fetch copies
  // only the breakpoints its rows hold.
  using CntT = typename std::conditional<(CAP < 256), uint8_t, uint16_t>::type;
  const size_t pi_bytes = ((size_t)L + 15) & ~(size_t)15;
  const size_t cnt_bytes = ((size_t)(L + 1) * 2 * sizeof(CntT) + 15) & ~(size_t)15;
  const bool ring = pi_bytes + cnt_bytes + (size_t)kWalkDepth * kWalkSlot <= INST_BYTES;
  const bool fin_smem = pi_bytes + cnt_bytes + (size_t)L * 8 <= INST_BYTES;
  uint8_t* pis = ring ? ws : a.out.pi + lo;
  CntT* cnts = reinterpret_cast<CntT*>(ws + pi_bytes);
  unsigned char* rbase = ws + pi_bytes + cnt_bytes;
  const bool infeasible = pmax == -INFINITY;
  int32_t status = SP_OK;
  __syncwarp(kFull);  // every lane is done with the rows and the scratch
  // one stage of the store into ring slot k % kWalkDepth (one commit group)
  // (only breakpoint pairs holding a breakpoint; a row of more than 64 is
  // searched in the store instead)
  auto fetch = [&](int k) {
    if (k >= 1) {
      unsigned char* sl = rbase + (size_t)(k % kWalkDepth) * kWalkSlot;
      const int2* er = g_ent + (size_t)(2 * k) * CAP;  // 16-B aligned: CAP is even
      const int fc = cnts[2 * k], fs = cnts[2 * k + 1];
      // (a row of odd count: its last breakpoint alone, never the unwritten slot after it)
      // (rows of odd count carry a padding entry: whole pairs; a lane with
      // nothing to copy points at the always-written row counts)
      const bool pc = fc <= 64 && 2 * lane < fc, ps = fs <= 64 && 2 * lane < fs;
      cp_async16_part(sl + 32 + lane * 16, pc ? (const void*)(er + 2 * lane) : (const void*)g_cnt, pc ? 16 : 0);
      cp_async16_part(sl + 32 + 512 + lane * 16, ps ? (const void*)(er + CAP + 2 * lane) : (const void*)g_cnt,
                      ps ? 16 : 0);
      if (lane == 0) cp_async16(sl, a.shifts + lo + k - 1);
    }
    cp_async_commit();
  };
  // the breakpoints of row `ent` (n of them) at or left of j, and the
  // stay_from of the last of them, with plain loads (32-ary search)
  auto search = [&](const int2* ent, int n, int j, int& c, int32_t& sf) {
    int lo_i = 0, hi_i = n;  // the count lies in [lo_i, hi_i]
    while (lo_i < hi_i) {
      const int span = hi_i - lo_i;
      const int step = (span + 32) / 33;
      const int p = lo_i + (lane + 1) * step - 1;
      const bool valid = p < hi_i;
      const int cc = __popc(__ballot_sync(kFull, valid && ent[p].x <= j));
      const int nv = __popc(__ballot_sync(kFull, valid));
      const int nlo = lo_i + cc * step;
      hi_i = cc < nv ? lo_i + (cc + 1) * step - 1 : hi_i;
      lo_i = nlo;
    }
    c = lo_i;
    sf = c > 0 ? ent[c - 1].y : kNoStay;
  };
  if (infeasible) {  // _infeasible: all-server placement, feasible = False
    for (int k = lane; k < L; k += 32) pis[k] = 0;
  } else {
    bool client = ec >= es;
    int j = (int)inf.w_eff;
    if (ring) {
      for (int k = lane; k < 2 * (L + 1); k += 32) cnts[k] = (CntT)g_cnt[k];
      __syncwarp(kFull);
      for (int d = 0; d < kWalkDepth; ++d) fetch(L - d);
    }
    for (int k = L; k >= 1; --k) {
      const size_t rr = (size_t)(2 * k + (client ? 0 : 1)) * CAP;
      StageShift sh;
      int n, c;
      int32_t sf;  // stay_from of the breakpoint covering j
      if (ring) {
        cp_async_wait<kWalkDepth - 1>();
        __syncwarp(kFull);
        const unsigned char* sl = rbase + (size_t)(k % kWalkDepth) * kWalkSlot;
        sh = *reinterpret_cast<const StageShift*>(sl);
        n = cnts[2 * k + (client ? 0 : 1)];
        if (n <= 64) {  // lane l holds breakpoints 2l and 2l + 1
          const int4 e = reinterpret_cast<const int4*>(sl + 32 + (client ? 0 : 512))[lane];
          c = __popc(__ballot_sync(kFull, 2 * lane < n && e.x <= j)) +
              __popc(__ballot_sync(kFull, 2 * lane + 1 < n && e.z <= j));
          sf = __shfl_sync(kFull, ((c - 1) & 1) ? e.w : e.y, ((c - 1) >> 1) & 31);
        } else {
          search(g_ent + rr, n, j, c, sf);
        }
        __syncwarp(kFull);  // the slot is refilled next
        fetch(k - kWalkDepth);
      } else {
        sh = a.shifts[lo + k - 1];
        n = g_cnt[2 * k + (client ? 0 : 1)];
        search(g_ent + rr, n, j, c, sf);
      }
      if (c == 0) {  // j left of the row's first breakpoint: unreachable
        status = SP_ERR_BACKTRACE;
        break;
      }
      const bool stay = j >= sf;
      if (lane == 0) pis[k - 1] = client ? 1 : 0;
      if (client) {
        j -= stay ? sh.i : sh.id;
        client = stay;
      } else {
        j -= stay ? sh.s : sh.su;
        client = !stay;
      }
      if (j < 0) {  // no predecessor reproduces the value (planner.py:168-169 / 177-178)
        status = SP_ERR_BACKTRACE;
        break;
      }
    }
    if (ring) cp_async_wait<0>();  // no copy may land after the ring is reused
  }
  __syncwarp(kFull);
  if (status != SP_OK) {
    if (lane == 0) a.out.status[inst] = status;
    return;
  }
  if (ring && fin_smem) {
    finish_policy_warp(a.in, inst, lo, L, pis, reinterpret_cast<double*>(rbase), a.out, infeasible, lane);
  } else if (lane == 0) {
    if (ring)
      for (int k = 0; k < L; ++k) a.out.pi[lo + k] = pis[k];
    sp_policies o = a.out;
    finish_policy(a.in, inst, lo, L, a.idx + lo, o, infeasible, false);
    a.out.status[inst] = SP_OK;
  }
}
