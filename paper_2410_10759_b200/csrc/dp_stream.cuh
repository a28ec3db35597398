// K2 for rows wider than one SM: the streaming kernel (rows in L2, bulk-copy
// windows, warp-specialised) and the experimental own-block kernel.
//
// Fragment of sp_planner.cu: included there inside namespace sp::(anonymous),
// after the declarations it uses; not a standalone header.
#pragma once

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

