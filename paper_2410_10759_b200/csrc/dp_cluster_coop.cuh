// K2 variants kept for parity coverage (forced with SPLITPLAN_DP_VARIANT):
// dp_cluster_kernel (rows in cluster DSMEM) and dp_coop_kernel (L2 rows via LDG).
//
// Fragment of sp_planner.cu: included there inside namespace sp::(anonymous),
// after the declarations it uses; not a standalone header.
#pragma once

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

