// K2 for rows wider than one SM: the streaming kernel (rows in L2, bulk-copy
// windows, warp-specialised).
//
// Fragment of sp_planner.cu: included there inside namespace sp::(anonymous),
// after the declarations it uses; not a standalone header.
#pragma once

// ---------------------------------------------------------------------------
// K2 streaming variant (rows longer than one SM's shared memory): a cluster
// of G CTAs shares one instance, CTA q owning NC chunks of CH = T*E columns.
// The rows live in global memory, DOUBLE-buffered (stage k reads buffer k%2
// and writes (k+1)%2), sized so the rows of every co-resident instance stay
// in L2.  Each CTA is warp-specialised:
//   * one producer warp fetches, for every chunk, the four predecessor windows
//     (C at i, S at i+d, S at s, C at s+u; CH values + 16 B, 16-B aligned)
//     with the bulk-copy engine (cp.async.bulk, completion on a `full`
//     mbarrier) into an NSLOT-deep ring of shared-memory slots;
//   * T compute threads read them with conflict-free LDS like the single-CTA
//     kernel, store the new cells straight to the next row buffer (coalesced
//     warp stores) and the back-pointer words with an L2 evict-first policy,
//     and release the slot on its `empty` mbarrier.
// Stages are ordered by per-CTA progress counters in shared memory, read by
// the other CTAs of the cluster through DSMEM, instead of a cluster-wide
// barrier: the producer of CTA q may start stage k once every CTA at or left
// of q finished stage k-1 (all reads go left: shifts are >= 0) and -- WAR on
// the buffer stage k overwrites, last read in stage k-1 -- every CTA finished
// stage k-1.

// shared-memory and cluster addressing
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t cluster_addr(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
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
// Progress counters: published with a release reduction, polled by the other
// CTAs of the cluster with relaxed loads (then an acquire fence) -- strong
// operations of cluster scope on both sides, i.e. synchronisation, not a race.
// (the counters only grow: a release max-reduction is the store)
__device__ __forceinline__ void st_cluster_release(uint32_t* p, uint32_t v) {
  asm volatile("red.release.cluster.shared::cta.max.u32 [%0], %1;" ::"r"(smem_addr(p)), "r"(v) : "memory");
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
